#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-ev}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -o gpurun_out/${TAG}_kernels python scripts/kernel_evidence.py > gpurun_out/${TAG}_ncu.log 2>&1
