"""One-line-per-launch summary of an ncu --set full report (read here, no GPU):
python scripts/ncu_summary.py gpurun_out/x.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {}
    for k in WANT:
        cands = [i for i, h in enumerate(hdr) if h == k]
        if cands:
            idx[k] = cands[0]
    name_i = hdr.index("Kernel Name")
    for r in rows[2:]:
        vals = {}
        for k, i in idx.items():
            v = r[i].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[i]
            if k == "gpu__time_duration.sum":
                x = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0) * x
            if k.startswith("dram__bytes") or k == "lts__t_bytes.sum":
                x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            vals[WANT[k]] = x
        vals.setdefault("dur_us", 0.0)
        nm = r[name_i].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[-48:]
        traffic = vals.get("dram_rd", 0) + vals.get("dram_wr", 0)
        gbs = traffic / (vals.get("dur_us", 1) * 1e-6) / 1e9
        print(f"{nm:48s} dur {vals.get('dur_us', 0):8.1f}us dram {traffic / 1e6:8.1f}MB ({gbs:6.0f} GB/s, "
              f"{vals.get('dram_pct', 0):4.1f}%) tensor {vals.get('tensor_pct', 0):4.1f}% sm {vals.get('sm_pct', 0):4.1f}% "
              f"occ {vals.get('occ_pct', 0):4.1f}% regs {vals.get('regs', 0):.0f} grid {vals.get('grid', 0):.0f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
