#!/bin/bash
# One GPU call: the whole -m gpu suite + smoke(), then the default bench line.
TAG=${TAG:-r2}
TAG=$TAG PYTEST_TIMEOUT=${PYTEST_TIMEOUT:-2400} bash scripts/gpu_tests.sh
timeout -s ABRT 900 python -X faulthandler bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
tail -c 3000 gpurun_out/${TAG}_bench.jsonl
