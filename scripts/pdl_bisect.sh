#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/pdl_bisect.log
T="tests/test_forward_gpu.py"
for m in ${MASKS:-15}; do
  AG_PDL_MASK=$m timeout 400 python -m pytest -x -q "$T" > gpurun_out/pdl_bisect_$m.log 2>&1
  echo "mask $m rc=$?" >> gpurun_out/pdl_bisect.log
  tail -1 gpurun_out/pdl_bisect_$m.log >> gpurun_out/pdl_bisect.log
done
if grep -q "mask 15 rc=0" gpurun_out/pdl_bisect.log; then
  for v in 11 15; do AG_PDL_MASK=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/pdl_bench_mask$v.log 2>&1; done
fi
