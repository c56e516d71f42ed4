#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/attn_ctas.log
C=chunk2048_on_8k,prefill_3072,prefill_6x512,chunk1024_on_15k
for n in 0 100000 296; do
  echo "== AG_ATTN_TILE_CTAS=$n" >> gpurun_out/attn_ctas.log
  AG_ATTN_TILE_CTAS=$n ATTN_CASES=$C timeout 300 python scripts/attn_bench.py 40 >> gpurun_out/attn_ctas.log 2>&1
done
NVCC_EXTRA="-DAG_ATTN_TIMELINE" python -c "from paper_2503_13737_b200 import build; build.build(force=True)" > /dev/null 2>&1
AG_ATTN_TILE_CTAS=100000 timeout 120 python scripts/attn_timeline.py chunk2048_on_8k >> gpurun_out/attn_ctas.log 2>&1
