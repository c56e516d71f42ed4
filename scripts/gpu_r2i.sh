#!/bin/bash
# TP tests after the OOM fix; AccelGen vs baselines on the B200 executor (refined policy); PDL mask-15 hang repro
timeout 1200 python -m pytest tests/test_tp_gpu.py -m gpu -q -s > gpurun_out/r2i_tp.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_tp.log
tail -3 gpurun_out/r2i_tp.log
RATE=8 bash scripts/gpu_policy_compare.sh
mkdir -p gpurun_out/r2i_policy8 && cp gpurun_out/policy/*.csv gpurun_out/policy/*.json gpurun_out/policy/*.log gpurun_out/r2i_policy8/ 2>/dev/null
tail -6 gpurun_out/r2i_policy8/run.log
AG_PDL_MASK=15 timeout 420 python bench.py --steps 5 --warmup 3 --ramp-s 40 --no-cpu-baseline > gpurun_out/r2i_pdl15.jsonl 2> gpurun_out/r2i_pdl15.err
echo "pdl15 rc=$?" >> gpurun_out/r2i_pdl15.err
tail -2 gpurun_out/r2i_pdl15.err
nvidia-smi --query-gpu=name,memory.used --format=csv >> gpurun_out/r2i_pdl15.err 2>&1
