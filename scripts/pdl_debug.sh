#!/bin/bash
mkdir -p gpurun_out
T="tests/test_forward_gpu.py::test_13b_shape_mixed_batch_two_layers"
AG_PDL_MASK=5 timeout 300 python -m pytest -x -q -s "$T" > gpurun_out/pdl_debug.log 2>&1
echo "rc=$?" >> gpurun_out/pdl_debug.log
