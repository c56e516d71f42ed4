#!/bin/bash
# One GPU call: bench lines at several (rate, steps) points; each line lands in gpurun_out/${TAG}_bench.jsonl.
# POINTS="rate:steps:ramp ..." (ramp empty = bench default)
TAG=${TAG:-r2}
mkdir -p gpurun_out/plan_cache
export AG_GEMM_PLAN_CACHE=gpurun_out/plan_cache  # autotune once per library build
for pt in ${POINTS:-"3:20:"}; do
  IFS=: read rate steps ramp <<< "$pt"
  extra=""
  [ -n "$ramp" ] && extra="--ramp-s $ramp"
  echo "== rate=$rate steps=$steps ramp=$ramp" >> gpurun_out/${TAG}_bench.log
  timeout ${BENCH_TIMEOUT:-900} python bench.py --rate $rate --steps $steps --warmup 3 $extra ${BENCH_ARGS} \
     > gpurun_out/${TAG}_one.out 2>> gpurun_out/${TAG}_bench.log
  echo "rc=$?" >> gpurun_out/${TAG}_bench.log
  tail -1 gpurun_out/${TAG}_one.out >> gpurun_out/${TAG}_bench.jsonl
done
