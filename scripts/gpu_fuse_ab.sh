#!/bin/bash
# Fused LayerNorm tail: GPU tests (whole -m gpu suite + smoke), in-chain A/B on the ablation probe
# batches (fused vs AG_FUSE_LN=0), then the default bench line.
TAG=${TAG:-r2fa}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
TAG=$TAG PYTEST_TIMEOUT=1500 bash scripts/gpu_tests.sh
for i in 1 2; do
  timeout 600 python scripts/ablate_probe.py fused >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
  AG_FUSE_LN=0 timeout 600 python scripts/ablate_probe.py unfused >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
done
AG_ABLATE=4 timeout 600 python scripts/ablate_probe.py fused_noLN >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
cat gpurun_out/${TAG}_ab.jsonl
if [ -z "$SKIP_BENCH" ]; then
timeout -s ABRT 900 python -X faulthandler bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench.jsonl').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','iter_slo_attainment','ms_per_step')}, d.get('e2e'), d.get('kernel_share'), d.get('forward_roofline'), d.get('pivot_forward'))"
fi
