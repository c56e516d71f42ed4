#!/bin/bash
# autotuner now times out-proj / FC2 with their consuming LayerNorm; in-chain plan check
timeout 1500 python scripts/plan_probe2.py > gpurun_out/r2n_plan_probe.jsonl 2> gpurun_out/r2n_plan_probe.err
echo "probe rc=$?" >> gpurun_out/r2n_plan_probe.err
AG_ABLATE=0 timeout 400 python scripts/ablate_probe.py a0 > gpurun_out/r2n_ablate.jsonl 2> gpurun_out/r2n_ablate.err
cat gpurun_out/r2n_plan_probe.jsonl gpurun_out/r2n_ablate.jsonl
