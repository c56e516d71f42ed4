#!/bin/bash
# in-chain time attribution: the same bench-like OPT-13B batches with one kernel class skipped at a time
export AG_GEMM_PLAN_CACHE=/tmp/ablate_plans_$$
: > gpurun_out/r2j_ablate.jsonl
for m in 0 4 1 2 8 0; do
  AG_ABLATE=$m timeout 600 python scripts/ablate_probe.py a$m >> gpurun_out/r2j_ablate.jsonl 2>> gpurun_out/r2j_ablate.err
done
AG_PDL=0 timeout 600 python scripts/ablate_probe.py nopdl >> gpurun_out/r2j_ablate.jsonl 2>> gpurun_out/r2j_ablate.err
AG_PDL=0 AG_ABLATE=4 timeout 600 python scripts/ablate_probe.py nopdl_a4 >> gpurun_out/r2j_ablate.jsonl 2>> gpurun_out/r2j_ablate.err
cat gpurun_out/r2j_ablate.jsonl
timeout 1200 python -m pytest tests/test_tp_gpu.py -m gpu -q -s > gpurun_out/r2j_tp.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tp.log
tail -3 gpurun_out/r2j_tp.log
RATE=8 bash scripts/gpu_policy_compare.sh
mkdir -p gpurun_out/r2j_policy8 && cp gpurun_out/policy/*.csv gpurun_out/policy/*.json gpurun_out/policy/*.log gpurun_out/r2j_policy8/ 2>/dev/null
tail -6 gpurun_out/r2j_policy8/run.log
# PDL mask-15 hang: which part of the serving loop triggers it (SIGABRT -> faulthandler traceback)
pdl() {  # tag, env, args
  env $2 timeout -s ABRT 240 python -X faulthandler bench.py --steps 3 --warmup 3 --ramp-s 20 --no-cpu-baseline $3 \
    > gpurun_out/r2j_pdl_$1.jsonl 2> gpurun_out/r2j_pdl_$1.err
  echo "$1 rc=$?" | tee -a gpurun_out/r2j_pdl_summary.txt
}
pdl m15_nopipe AG_PDL_MASK=15 --no-pipeline
pdl m15_rate1 AG_PDL_MASK=15 "--rate 1"
pdl m7 AG_PDL_MASK=7 ""
pdl m15 AG_PDL_MASK=15 ""
nvidia-smi --query-gpu=name,memory.used --format=csv >> gpurun_out/r2j_pdl_summary.txt 2>&1
