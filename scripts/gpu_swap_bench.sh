#!/bin/bash
# Swap path tests, then the default bench line (host time of the swap path: swap_host, host_ms_per_step).
TAG=${TAG:-r2sw}
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_forward_gpu.py -k "swap" -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
timeout -s ABRT 900 python -X faulthandler bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench.jsonl').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','iter_slo_attainment','ms_per_step','preemptions_in_window','swap_gb_total')}, d.get('e2e'), d.get('host_ms_per_step'), d.get('swap_host'), d.get('kernel_share'))"
