#!/bin/bash
# in-chain time attribution (ablation) + PDL mask-15 hang on a plain forward loop (no engine)
export AG_GEMM_PLAN_CACHE=/tmp/ablate_plans_$$
: > gpurun_out/r2k_ablate.jsonl
run() { env $2 timeout -s ABRT ${3:-400} python -X faulthandler scripts/ablate_probe.py $1 >> gpurun_out/r2k_ablate.jsonl 2>> gpurun_out/r2k_ablate_$1.err; echo "$1 rc=$?" >> gpurun_out/r2k_summary.txt; }
run a0 AG_ABLATE=0
run a4 AG_ABLATE=4
run a1 AG_ABLATE=1
run a2 AG_ABLATE=2
run a8 AG_ABLATE=8
run a0b AG_ABLATE=0
run nopdl AG_PDL=0
run nopdl_a4 "AG_PDL=0 AG_ABLATE=4"
run m15 AG_PDL_MASK=15 200
run m15_det "AG_PDL_MASK=15 AG_DETERMINISTIC=1" 200
cat gpurun_out/r2k_ablate.jsonl gpurun_out/r2k_summary.txt
