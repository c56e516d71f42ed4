#!/bin/bash
# attention iteration: parity tests (debug build: mbarrier waits trap quickly), attn_bench, timeline
mkdir -p gpurun_out; rm -f gpurun_out/attn_round.log
NVCC_EXTRA="-DAG_DEBUG_MBAR $B_FLAGS" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 300 python -m pytest -q -x tests/test_kernels_gpu.py -k "attention or attn" > gpurun_out/attn_round_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/attn_round_tests.log
NVCC_EXTRA="$B_FLAGS" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 300 python -m pytest -q -x tests/test_forward_gpu.py -k "13b or 175b or config1" >> gpurun_out/attn_round_tests.log 2>&1; echo "fwd tests rc=$?" >> gpurun_out/attn_round_tests.log
ATTN_CASES=${ATTN_CASES_R:-chunk2048_on_8k,prefill_3072,prefill_6x512,chunk1024_on_15k,mixed,live_dec40_chunk280_on1200,live_dec40_fresh300} timeout 300 python scripts/attn_bench.py 40 >> gpurun_out/attn_round.log 2>&1
NVCC_EXTRA="-DAG_ATTN_TIMELINE $B_FLAGS" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
for c in chunk2048_on_8k prefill_6x512; do timeout 120 python scripts/attn_timeline.py $c >> gpurun_out/attn_round.log 2>&1; done
