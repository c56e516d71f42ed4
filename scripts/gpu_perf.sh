#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-perf}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python scripts/attn_bench.py > gpurun_out/${TAG}_attn.jsonl 2>&1
timeout 600 python scripts/gemm_sweep.py > gpurun_out/${TAG}_gemm.jsonl 2>&1
