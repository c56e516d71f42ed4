#!/bin/bash
# end-of-round evidence: whole -m gpu suite + smoke, the default bench line, ncu launch list of the
# timed windows + --set full of the first attention / GEMM launches, TP=2 bench plumbing (host backend)
TAG=${TAG:-r2end}
TAG=$TAG PYTEST_TIMEOUT=1800 bash scripts/gpu_tests.sh
timeout -s ABRT 900 python -X faulthandler bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
TAG=$TAG bash scripts/gpu_r2_evidence.sh
