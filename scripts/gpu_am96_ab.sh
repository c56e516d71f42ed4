#!/bin/bash
# 96-row A stages for 65..96-row GEMMs: kernel tests, then in-chain A/B (autotune with / without am=96).
TAG=${TAG:-r2am}
timeout 600 python -m pytest tests/test_kernels_gpu.py -k "small_m" tests/test_forward_gpu.py -k "small_m or full_depth or config1" -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; grep -E "FAILED|Error" gpurun_out/${TAG}_pytest.log | head -5
for i in 1 2; do
  timeout 600 python scripts/ablate_probe.py am96 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
  AG_TUNE_NO_AM96=1 timeout 600 python scripts/ablate_probe.py no_am96 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
done
cat gpurun_out/${TAG}_ab.jsonl; tail -3 gpurun_out/${TAG}_ab.err
