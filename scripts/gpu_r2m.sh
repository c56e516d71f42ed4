#!/bin/bash
# (1) default PDL scheme restored: probe timing; (2) mask 15 with stream-K replaced by classic 6-way
# atomic split-K (grid < all SMs): does the hang follow stream-K?; (3) sustained GEMM vs cuBLAS
export AG_GEMM_PLAN_CACHE=/tmp/pc_$$
: > gpurun_out/r2m_ablate.jsonl; : > gpurun_out/r2m_summary.txt
run() { env $2 timeout -s ABRT ${3:-400} python -X faulthandler scripts/ablate_probe.py $1 >> gpurun_out/r2m_ablate.jsonl 2>> gpurun_out/r2m_ablate_$1.err; echo "$1 rc=$?" >> gpurun_out/r2m_summary.txt; }
run a0 AG_ABLATE=0
python - <<PY
import json, pathlib
src = pathlib.Path("/tmp/pc_$$"); dst = pathlib.Path("/tmp/pcns_$$"); dst.mkdir(exist_ok=True)
for f in src.glob("*.json"):
    rows = json.loads(f.read_text())
    for r in rows:
        if r[3] % 100 == 99:
            r[3] = r[3] - 99 + 6
    (dst / f.name).write_text(json.dumps(rows))
    print("rewrote", f.name)
PY
run a0_ns "AG_GEMM_PLAN_CACHE=/tmp/pcns_$$"
run m15_ns "AG_GEMM_PLAN_CACHE=/tmp/pcns_$$ AG_PDL_MASK=15" 200
run a0b AG_ABLATE=0
timeout 900 python scripts/gemm_sustained.py 1536 > gpurun_out/r2m_gemm_sustained.jsonl 2> gpurun_out/r2m_gemm_sustained.err
timeout 600 python scripts/gemm_sustained.py 512 >> gpurun_out/r2m_gemm_sustained.jsonl 2>> gpurun_out/r2m_gemm_sustained.err
cat gpurun_out/r2m_ablate.jsonl gpurun_out/r2m_summary.txt gpurun_out/r2m_gemm_sustained.jsonl
