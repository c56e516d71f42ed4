#!/bin/bash
TAG=${TAG:-r2pf}
timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_kernels_gpu.py -k "swap" -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; grep -E "FAILED|Error" gpurun_out/${TAG}_pytest.log | head -5
timeout -s ABRT 900 python -X faulthandler bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench.jsonl').read().strip().splitlines()[-1])
print(round(d['value']), d['e2e'], round(d['iter_slo_attainment'],4), d['preemptions_in_window'], d['host_ms_per_step'], d['swap_host'])"
