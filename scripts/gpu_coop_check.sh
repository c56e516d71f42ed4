#!/bin/bash
# Cooperative launch of the fused-LayerNorm GEMMs: forward tests, ncu --set full replay of fused GEMMs
# (failed with LaunchFailed without the cooperative attribute), in-chain A/B.
TAG=${TAG:-r2co}
timeout 900 python -m pytest tests/test_forward_gpu.py -k "split_k or full_depth or config1" tests/test_pdl_gpu.py -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
grep -E "FAILED|Error" gpurun_out/${TAG}_pytest.log | head -5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm --launch-skip 40 --launch-count 8 \
  -o gpurun_out/${TAG}_fused_full python tests/helpers/pdl_atomic_stress.py > gpurun_out/${TAG}_ncu.out 2>&1
echo "ncu rc=$?"; tail -4 gpurun_out/${TAG}_ncu.out
for i in 1 2; do
  timeout 600 python scripts/ablate_probe.py fused >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
  AG_FUSE_LN=0 timeout 600 python scripts/ablate_probe.py unfused >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
done
cat gpurun_out/${TAG}_ab.jsonl; tail -3 gpurun_out/${TAG}_ab.err
