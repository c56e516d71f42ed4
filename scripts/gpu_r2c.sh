#!/bin/bash
# profiler (prefill + mixed sweep, extended fit) then bench stability: 20 vs 200 windows on the new profile
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
timeout 900 python -m paper_2503_13737_b200.profiler --out gpurun_out/opt13b_b200_tp1.json --kv-gb 153 > gpurun_out/r2c_profiler.log 2>&1
echo "profiler rc=$?" >> gpurun_out/r2c_profiler.log
P=gpurun_out/opt13b_b200_tp1.json
[ -f $P ] || P=profiles/opt13b_b200_tp1.json
for st in 20 200; do
  timeout 1500 python bench.py --steps $st --warmup 3 --profile $P > gpurun_out/r2c_bench_$st.out 2> gpurun_out/r2c_bench_$st.err
  echo "rc=$?" >> gpurun_out/r2c_bench_$st.err
done
tail -c 400 gpurun_out/r2c_bench_200.out
