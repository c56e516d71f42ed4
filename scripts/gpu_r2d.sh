#!/bin/bash
# new GPU tests (async steps, swap ring) + bench 20 and 200 windows with the pipelined engine
free -g > gpurun_out/r2d_free.txt; nproc >> gpurun_out/r2d_free.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1
timeout 900 python -m pytest tests/test_async_gpu.py tests/test_forward_gpu.py -k "async or swap or pipelined or config1" -m gpu -q -s -x > gpurun_out/r2d_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
for st in 20 200; do
  ( while sleep 20; do free -m | awk '/Mem/{print $3, $7}' >> gpurun_out/r2d_mem_$st.txt; done ) & MP=$!
  timeout 1500 python bench.py --steps $st --warmup 3 > gpurun_out/r2d_bench_$st.out 2> gpurun_out/r2d_bench_$st.err
  echo "rc=$?" >> gpurun_out/r2d_bench_$st.err
  kill $MP
done
tail -3 gpurun_out/r2d_pytest.log; tail -c 300 gpurun_out/r2d_bench_20.out
