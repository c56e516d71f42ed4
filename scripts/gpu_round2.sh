#!/bin/bash
# One GPU call: -m gpu suite + smoke + default bench line (+ optional launch list).  Logs in gpurun_out/.
TAG=${TAG:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.used --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
lscpu | head -20 > gpurun_out/${TAG}_lscpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout ${PYTEST_TIMEOUT:-2400} python -m pytest ${SEL:-tests} -m gpu -q -s --durations=30 ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
fi
if [ -z "$SKIP_BENCH" ]; then
timeout ${BENCH_TIMEOUT:-1200} python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.out 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
fi
tail -3 gpurun_out/${TAG}_pytest_gpu.log 2>/dev/null; tail -c 600 gpurun_out/${TAG}_bench.out 2>/dev/null
