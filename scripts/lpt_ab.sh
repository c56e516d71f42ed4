#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/lpt_ab.log
timeout 300 python -m pytest -q -x tests/test_kernels_gpu.py -k "attention or attn" > gpurun_out/lpt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lpt_tests.log
C=decode_var64,live_var48_chunk200,mixed,mixed_small_prompts,live_dec40_chunk280_on1200,decode_256x2k
for rep in 1 2; do
  echo "== LPT" >> gpurun_out/lpt_ab.log; ATTN_CASES=$C python scripts/attn_bench.py 40 >> gpurun_out/lpt_ab.log 2>&1
  echo "== no LPT" >> gpurun_out/lpt_ab.log; AG_ATTN_NO_LPT=1 ATTN_CASES=$C python scripts/attn_bench.py 40 >> gpurun_out/lpt_ab.log 2>&1
done
