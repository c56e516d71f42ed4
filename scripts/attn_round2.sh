#!/bin/bash
# attention change check: parity (debug build), forward tests, attn_bench mixed cases, default bench
mkdir -p gpurun_out; rm -f gpurun_out/attn_round2.log
NVCC_EXTRA="-DAG_DEBUG_MBAR" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 300 python -m pytest -q -x tests/test_kernels_gpu.py -k "attention or attn" > gpurun_out/attn_round2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/attn_round2_tests.log
python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 600 python -m pytest -q -x tests/test_forward_gpu.py >> gpurun_out/attn_round2_tests.log 2>&1; echo "fwd tests rc=$?" >> gpurun_out/attn_round2_tests.log
ATTN_CASES=chunk2048_on_8k,prefill_3072,prefill_6x512,mixed,mixed_small_prompts,live_dec40_chunk280_on1200,live_dec40_fresh300,live_var48_chunk200 timeout 300 python scripts/attn_bench.py 40 >> gpurun_out/attn_round2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/attn_round2_bench.log 2>&1
