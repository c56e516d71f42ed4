#!/bin/bash
# One GPU call: parity tests, smoke, a default bench line, the ncu launch list of the timed steps and
# one --set full capture of the attention and GEMM kernels inside the timed region (AG_NCU_TIMED=1:
# cudaProfilerStart/Stop around the K timed steps). Run under gpurun; everything lands in gpurun_out/.
mkdir -p gpurun_out/plan_cache
cp .plan_cache/* gpurun_out/plan_cache/ 2>/dev/null
export AG_GEMM_PLAN_CACHE=gpurun_out/plan_cache  # autotune once per library build (bench/ncu runs reuse it)
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | head -20 >> gpurun_out/${TAG}_nproc.txt
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
fi
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
if [ -z "$SKIP_NCU" ]; then
AG_NCU_TIMED=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
AG_NCU_TIMED=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"mixed_attention" -c 2 -o gpurun_out/${TAG}_attn_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_attn.log 2>&1
AG_NCU_TIMED=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"gemm" -c 5 -o gpurun_out/${TAG}_gemm_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_gemm.log 2>&1
fi
ls -la gpurun_out
