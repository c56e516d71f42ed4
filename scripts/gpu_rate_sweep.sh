#!/bin/bash
# rate sweep of the pipelined bench (20 windows each): the highest rate with >= 95% iteration-SLO attainment
TAG=${TAG:-r2e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
mkdir -p gpurun_out/plan_cache
export AG_GEMM_PLAN_CACHE=gpurun_out/plan_cache
for r in ${RATES:-3.5 4 5 6}; do
  timeout -s ABRT 600 python -X faulthandler bench.py --rate $r --steps 20 --warmup 3 ${BENCH_ARGS} --no-cpu-baseline > gpurun_out/${TAG}_rate_$r.out 2> gpurun_out/${TAG}_rate_$r.err
  echo "rate $r rc=$?" >> gpurun_out/${TAG}_sweep.log
  tail -1 gpurun_out/${TAG}_rate_$r.out >> gpurun_out/${TAG}_sweep.jsonl
done
cat gpurun_out/${TAG}_sweep.log
