#!/bin/bash
# PDL default mask 15 + fenced atomic epilogues: tests, then the higher-rate sweep (also a long no-hang run)
timeout 1200 python -m pytest tests/test_pdl_gpu.py -m gpu -q -s > gpurun_out/r2r_pdl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_pdl_tests.log
tail -3 gpurun_out/r2r_pdl_tests.log
TAG=r2r RATES="4 5 5.5 6 7" bash scripts/gpu_rate_sweep.sh
