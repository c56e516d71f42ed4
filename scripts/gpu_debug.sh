#!/bin/bash
mkdir -p gpurun_out
AG_DEBUG_SYNC=1 timeout 600 python -m pytest tests/test_forward_gpu.py -q -x -k 13b > gpurun_out/dbg_13b.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/dbg_all.log 2>&1
