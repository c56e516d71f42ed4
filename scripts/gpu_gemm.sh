#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-g}
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "gemm" > gpurun_out/${TAG}_pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_gemm.log
timeout 900 python scripts/gemm_sweep.py ${MS:-256,512,1024,2048,3072} > gpurun_out/${TAG}_gemm.jsonl 2>&1
