#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/row_split.log
C=decode_256x2k,decode_1x100k,live_dec40,live_dec40_chunk280_on1200,mixed,mixed_small_prompts,live_dec60_chunk64_on510
for cfg in ${CFGS:-"24 512" "12 512" "16 512" "12 1024" "8 1024"}; do
  set -- $cfg
  echo "== warps $1 min $2" >> gpurun_out/row_split.log
  AG_ATTN_ROW_WARPS=$1 AG_ATTN_ROW_MIN=$2 ATTN_CASES=$C timeout 300 python scripts/attn_bench.py 40 >> gpurun_out/row_split.log 2>&1
done
