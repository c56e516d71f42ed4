"""In-chain GEMM plan check: the OPT-13B forward (40 layers) on bench-like batches with the autotuned
plan table, then with the out-proj / FC2 plan of the batch's M bucket forced to each candidate (the
rest of the table unchanged).  Forward device time per candidate; compares what the autotuner picked
with what is fastest inside the real launch chain.  python scripts/plan_probe2.py -> JSON lines."""
import ctypes as C
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from ablate_probe import build  # noqa: E402
from paper_2503_13737_b200 import _lib, model as Mo  # noqa: E402
from paper_2503_13737_b200.executor import CudaExecutor  # noqa: E402

rng = np.random.default_rng(1)
BATCHES = {
    "decode60_chunk30": [(int(c), 1) for c in rng.integers(300, 4000, 60)] + [(0, 30)],
    "chunk448_dec64": [(2048, 448)] + [(int(c), 1) for c in rng.integers(300, 4000, 64)],
    "chunk1024": [(3000, 1024)],
    "pivot1536": [(4096, 1520)] + [(int(c), 1) for c in rng.integers(300, 4000, 16)],
}
KINDS = ("qkv", "out", "fc1", "fc2", "lm_head")
CANDS = [(256, 1, 256), (256, 2, 256), (256, 3, 256), (256, 99, 256), (128, 99, 256), (256, 1, 128),
         (256, 2, 128), (256, 99, 128), (128, 99, 128), (128, 1, 128), (256, 6, 64), (256, 99, 64)]


def main():
    cfg = Mo.opt_13b(max_positions=8192)
    need = max(sum((c + n + 31) // 32 for c, n in segs) for segs in BATCHES.values()) + 8
    ex = CudaExecutor(cfg, need, max_tokens=1536, max_seqs=256, autotune=True)
    base = ex.gemm_plans()  # (kind, m_bucket, bn, ks, am)
    print(json.dumps({"autotuned": [f"{k}:{mb}:{bn}x{ks}a{am}" for k, mb, bn, ks, am in base]}), flush=True)

    def install(kind, mb, plan):
        rows = []
        for k, b, bn, ks, am in base:
            if k == kind and b == mb:
                bn, ks, am = plan
            rows.append([KINDS.index(k), b, bn, ks + 100 * am])
        buf = (C.c_int32 * (4 * len(rows)))(*[x for r in rows for x in r])
        _lib.check(ex.lib.ag_model_set_gemm_plans(ex.handle, buf, len(rows)))

    def timed(b):
        for _ in range(2):
            ex.execute(b)
        ts = sorted(ex.execute(b).device_s for _ in range(7))
        return round(ts[3] * 1e3, 3)

    for name, segs in BATCHES.items():
        b, _ = build(segs, cfg, 0)
        M = int(b.cu_q[-1])
        bucket = next(mb for k, mb, *_ in base if k == "out" and (M <= mb or mb == max(x[1] for x in base)))
        install("out", bucket, next((bn, ks, am) for k, mb, bn, ks, am in base if k == "out" and mb == bucket))
        row = {"batch": name, "M": M, "bucket": bucket, "autotuned_ms": timed(b),
               "picked": {k: f"{bn}x{ks}a{am}" for k, mb, bn, ks, am in base if mb == bucket}}
        for kind in ("out", "fc2"):
            res = {}
            for plan in CANDS:
                bn, ks, am = plan
                if am < 128 and M > am:
                    continue
                try:
                    install(kind, bucket, plan)
                    res[f"{bn}x{ks}a{am}"] = timed(b)
                except Exception as e:  # noqa: BLE001
                    res[f"{bn}x{ks}a{am}"] = str(e)[:60]
            install(kind, bucket, next((bn, ks, am) for k, mb, bn, ks, am in base if k == kind and mb == bucket))
            row[kind] = res
        print(json.dumps(row), flush=True)
    ex.close()


if __name__ == "__main__":
    main()
