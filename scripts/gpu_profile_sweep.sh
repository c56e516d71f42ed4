#!/bin/bash
# Re-measure the B200 cost model (profiler) with the current kernels, then sweep arrival rates on it.
mkdir -p gpurun_out/plan_cache
cp .plan_cache/* gpurun_out/plan_cache/ 2>/dev/null
export AG_GEMM_PLAN_CACHE=gpurun_out/plan_cache
TAG=${TAG:-ps}
timeout 900 python -m paper_2503_13737_b200.profiler --out gpurun_out/${TAG}_opt13b_b200_tp1.json > gpurun_out/${TAG}_profiler.log 2>&1
cp gpurun_out/${TAG}_opt13b_b200_tp1.json profiles/opt13b_b200_tp1.json 2>/dev/null
for r in ${RATES:-6 8 10 12 14}; do
  timeout 400 python bench.py --steps ${STEPS:-100} --warmup 5 --rate $r --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_rate$r.json
done
