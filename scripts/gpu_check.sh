#!/bin/bash
# One GPU call: parity tests, smoke, a default bench line, the ncu launch list and one full capture
# of the GEMM and the attention kernel. Run under gpurun; everything lands in gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | head -20 >> gpurun_out/${TAG}_nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"gemm_bf16|mixed_attention|attn_combine|layernorm|embed_kernel|argmax|splitk|kv_append" \
  -s 2000 -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 4 --warmup 1 --ramp-s 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16" -s 800 -c 3 \
  -o gpurun_out/${TAG}_gemm_full python bench.py --steps 3 --warmup 1 --ramp-s 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mixed_attention" -s 200 -c 2 \
  -o gpurun_out/${TAG}_attn_full python bench.py --steps 3 --warmup 1 --ramp-s 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_attn.log 2>&1
fi
ls -la gpurun_out
