#!/bin/bash
# One GPU call: the whole -m gpu suite (per-test durations) + smoke().  Logs land in gpurun_out/.
TAG=${TAG:-r2}
SEL=${SEL:-tests}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.used --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout ${PYTEST_TIMEOUT:-2400} python -m pytest $SEL -m gpu -q -s --durations=25 ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
if [ -z "$SKIP_SMOKE" ]; then
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
fi
tail -3 gpurun_out/${TAG}_pytest_gpu.log
