#!/bin/bash
# PDL trigger-after-wait invariant: the round-2 hang cases (norms early-launched / skipped behind a
# stream-K GEMM) must now complete; then in-chain timing with norms early-launched
export AG_GEMM_PLAN_CACHE=/tmp/ablate_plans_$$
: > gpurun_out/r2l_ablate.jsonl; : > gpurun_out/r2l_summary.txt
run() { env $2 timeout -s ABRT ${3:-400} python -X faulthandler scripts/ablate_probe.py $1 >> gpurun_out/r2l_ablate.jsonl 2>> gpurun_out/r2l_ablate_$1.err; echo "$1 rc=$?" >> gpurun_out/r2l_summary.txt; }
run a0 AG_ABLATE=0
run m15 AG_PDL_MASK=15 200
run m15_a4 "AG_PDL_MASK=15 AG_ABLATE=4" 200
run a4 AG_ABLATE=4 200
run m15_a1 "AG_PDL_MASK=15 AG_ABLATE=1" 200
run m15_a2 "AG_PDL_MASK=15 AG_ABLATE=2" 200
run nopdl AG_PDL=0
run m15b AG_PDL_MASK=15 200
AG_PDL_MASK=15 timeout -s ABRT 400 python -X faulthandler bench.py --steps 10 --warmup 3 --ramp-s 60 --no-cpu-baseline > gpurun_out/r2l_bench_m15.jsonl 2> gpurun_out/r2l_bench_m15.err
echo "bench m15 rc=$?" >> gpurun_out/r2l_summary.txt
timeout 900 python -m pytest tests/test_pdl_gpu.py tests/test_forward_gpu.py -m gpu -q -x > gpurun_out/r2l_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2l_summary.txt
cat gpurun_out/r2l_ablate.jsonl gpurun_out/r2l_summary.txt
