#!/bin/bash
# LayerNorm-in-consumer-prologue: forward tests that exercise it, then the in-chain A/B (fused vs AG_FUSE_LN=0).
TAG=${TAG:-r2pa}
timeout 900 python -m pytest tests/test_forward_gpu.py -k "split_k or full_depth or 175b or config1" tests/test_pdl_gpu.py -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
grep -E "FAILED|Error" gpurun_out/${TAG}_pytest.log | head -5
for i in 1 2; do
  timeout 600 python scripts/ablate_probe.py fused >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
  AG_FUSE_LN=0 timeout 600 python scripts/ablate_probe.py unfused >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
done
cat gpurun_out/${TAG}_ab.jsonl; tail -3 gpurun_out/${TAG}_ab.err
