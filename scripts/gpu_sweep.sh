#!/bin/bash
# arrival-rate sweep of bench.py (no CPU baseline) + the profiler sweep
mkdir -p gpurun_out/plan_cache
cp .plan_cache/* gpurun_out/plan_cache/ 2>/dev/null
export AG_GEMM_PLAN_CACHE=gpurun_out/plan_cache  # autotune once per library build (bench/ncu runs reuse it)
TAG=${TAG:-sw}
for r in ${RATES:-6 12 24 48}; do
  timeout 400 python bench.py --steps ${STEPS:-100} --warmup 5 --rate $r --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_rate$r.json
done
