#!/bin/bash
# attention variants: tests + attn_bench + timeline per build flag set
mkdir -p gpurun_out; rm -f gpurun_out/attn_var.log
C=chunk2048_on_8k,prefill_3072,prefill_6x512,chunk1024_on_15k,mixed
for F in "" "-DAG_ATTN_EXP_POLY=4" "-DAG_ATTN_Q_TMEM" "-DAG_ATTN_Q_TMEM -DAG_ATTN_EXP_POLY=4" "-DAG_ATTN_Q_TMEM -DAG_ATTN_EXP_POLY=3"; do
  NVCC_EXTRA="$F" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
  echo "== [$F]" >> gpurun_out/attn_var.log
  timeout 300 python -m pytest -q -x tests/test_kernels_gpu.py -k "attention or attn" 2>&1 | tail -1 >> gpurun_out/attn_var.log
  ATTN_CASES=$C python scripts/attn_bench.py 40 >> gpurun_out/attn_var.log 2>&1
  NVCC_EXTRA="-DAG_ATTN_TIMELINE $F" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
  python scripts/attn_timeline.py chunk2048_on_8k 2>&1 | grep -E "cycles|per-tile" >> gpurun_out/attn_var.log
done
