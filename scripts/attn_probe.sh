#!/bin/bash
# Build a probe variant of the library (softmax skipped) and time the tile path: pipeline bound
mkdir -p gpurun_out
ATTN_CASES=chunk2048_on_8k,prefill_3072 python scripts/attn_bench.py 40 > gpurun_out/probe_base.jsonl 2>&1
NVCC_EXTRA=-DAG_ATTN_PIPE_PROBE python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > gpurun_out/probe_build.log 2>&1
ATTN_CASES=chunk2048_on_8k,prefill_3072 python scripts/attn_bench.py 40 > gpurun_out/probe_skip.jsonl 2>&1
