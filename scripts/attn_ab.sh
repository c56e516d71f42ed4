#!/bin/bash
# A/B of an attention variant: parity tests on the default build, then attn_bench default vs $B_FLAGS.
mkdir -p gpurun_out; rm -f gpurun_out/attn_ab.log
C=${ATTN_CASES_AB:-chunk2048_on_8k,prefill_3072,prefill_6x512,chunk1024_on_15k,mixed,live_dec40_chunk280_on1200}
timeout 600 python -m pytest -q -x tests/test_kernels_gpu.py -k "attention or attn" > gpurun_out/attn_ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/attn_ab_tests.log
echo "== default" >> gpurun_out/attn_ab.log
ATTN_CASES=$C python scripts/attn_bench.py 40 >> gpurun_out/attn_ab.log 2>&1
NVCC_EXTRA="$B_FLAGS" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
echo "== $B_FLAGS" >> gpurun_out/attn_ab.log
ATTN_CASES=$C python scripts/attn_bench.py 40 >> gpurun_out/attn_ab.log 2>&1
