#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/probe3.log
tl() {
  NVCC_EXTRA="-DAG_ATTN_TIMELINE $2" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > gpurun_out/probe_build_$1.log 2>&1
  for c in ${CASES:-chunk2048_on_8k prefill_3072}; do
    echo "== $1 ($2)" >> gpurun_out/probe3.log
    python scripts/attn_timeline.py $c >> gpurun_out/probe3.log 2>&1
  done
}
tl base ""
tl sbuf2 "-DAG_ATTN_SBUF=2"
