#!/bin/bash
# Timing probes of the tile path (results are wrong by construction; timing only):
#   base | no softmax | no softmax + no P.V | no softmax + no TMA | no softmax + no TMA + no P.V
mkdir -p gpurun_out
C=chunk2048_on_8k,prefill_3072
run() {  # $1 tag, $2 flags
  NVCC_EXTRA="$2" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > gpurun_out/probe_build_$1.log 2>&1
  echo "== $1 ($2)" >> gpurun_out/probe.log
  ATTN_CASES=$C python scripts/attn_bench.py 40 >> gpurun_out/probe.log 2>&1
}
rm -f gpurun_out/probe.log
run base ""
run nosm "-DAG_ATTN_PIPE_PROBE"
run nosm_nopv "-DAG_ATTN_PIPE_PROBE -DAG_ATTN_PROBE_NOPV"
run nosm_notma "-DAG_ATTN_PIPE_PROBE -DAG_ATTN_PROBE_NOTMA"
run nosm_notma_nopv "-DAG_ATTN_PIPE_PROBE -DAG_ATTN_PROBE_NOTMA -DAG_ATTN_PROBE_NOPV"
run notma "-DAG_ATTN_PROBE_NOTMA"
