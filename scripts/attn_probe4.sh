#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/probe4.log
C=chunk2048_on_8k,prefill_3072
run() {
  NVCC_EXTRA="$2" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
  echo "== $1 ($2)" >> gpurun_out/probe4.log
  ATTN_CASES=$C python scripts/attn_bench.py 40 >> gpurun_out/probe4.log 2>&1
}
run base ""
run noexp "-DAG_ATTN_PROBE_NOEXP"
run nolds "-DAG_ATTN_PROBE_NOLDS"
run noexp_nolds "-DAG_ATTN_PROBE_NOEXP -DAG_ATTN_PROBE_NOLDS"
