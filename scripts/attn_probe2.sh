#!/bin/bash
mkdir -p gpurun_out
C=chunk2048_on_8k,prefill_3072,prefill_6x512,decode_256x2k,mixed
run() {
  NVCC_EXTRA="$2" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > gpurun_out/probe_build_$1.log 2>&1
  echo "== $1 ($2)" >> gpurun_out/probe2.log
  ATTN_CASES=$C python scripts/attn_bench.py 40 >> gpurun_out/probe2.log 2>&1
}
rm -f gpurun_out/probe2.log
P="-DAG_ATTN_PIPE_PROBE -DAG_ATTN_PROBE_NOTMA -DAG_ATTN_PROBE_NOPV"
run base ""
run skeleton "$P -DAG_ATTN_PROBE_NOS"
run s_only "$P"
