#!/bin/bash
# Load sweep + ncu evidence for profiles/ (run under gpurun)
set -x
mkdir -p gpurun_out
for r in 3 6 9; do
  timeout 300 python bench.py --steps 60 --warmup 3 --rate $r --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_rate$r.json
done
# launch list of our kernels (cold, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_bf16|mixed_attention|attn_combine|layernorm|embed_kernel|argmax" -s 1500 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 1 --ramp-s 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
# one full capture of the top kernels
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16" -s 600 -c 2 -o gpurun_out/gemm_full python bench.py --steps 3 --warmup 1 --ramp-s 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mixed_attention" -s 150 -c 2 -o gpurun_out/attn_full python bench.py --steps 3 --warmup 1 --ramp-s 3 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
