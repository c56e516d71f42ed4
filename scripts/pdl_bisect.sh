#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/pdl_bisect.log
T="tests/test_forward_gpu.py::test_13b_shape_mixed_batch_two_layers"
for m in ${MASKS:-3 5 6 9 10 12}; do
  AG_PDL_MASK=$m timeout 100 python -m pytest -x -q "$T" > gpurun_out/pdl_bisect_$m.log 2>&1
  echo "mask $m rc=$?" >> gpurun_out/pdl_bisect.log
done
