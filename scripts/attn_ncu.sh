#!/bin/bash
# ncu --set full (source-level) of the attention kernel on one prefill case.
mkdir -p gpurun_out
CASE=${CASE:-chunk2048_on_8k}
ATTN_CASES=$CASE timeout 900 ncu --set full --clock-control none --import-source on -k regex:mixed_attention -s 3 -c 1 \
  -o gpurun_out/attn_${CASE}_full python scripts/attn_bench.py 40 > gpurun_out/attn_ncu_${CASE}.log 2>&1
echo "rc=$?" >> gpurun_out/attn_ncu_${CASE}.log
