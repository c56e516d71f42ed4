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
