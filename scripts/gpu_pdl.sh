#!/bin/bash
# PDL A/B: GPU parity tests with PDL on, autotune table and bench with AG_PDL=0 / 1.
mkdir -p gpurun_out
T=${TAG:-pdl}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
for v in 0 1; do
  AG_PDL=$v timeout 600 python scripts/autotune_log.py > gpurun_out/${T}_autotune_pdl$v.txt 2>&1
  AG_PDL=$v timeout 600 python bench.py --steps 120 --no-cpu-baseline > gpurun_out/${T}_bench_pdl$v.log 2>&1
done
