#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-a}
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "attention" > gpurun_out/${TAG}_pytest_attn.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_attn.log
timeout 600 python -m pytest tests/test_forward_gpu.py -q > gpurun_out/${TAG}_pytest_fwd.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_fwd.log
timeout 600 python scripts/attn_bench.py 40 scripts/attn_cases_r8.json > gpurun_out/${TAG}_attn.jsonl 2>&1
