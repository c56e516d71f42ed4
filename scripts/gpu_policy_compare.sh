#!/bin/bash
# AccelGen vs the SPEC baselines on the B200 executor (device clock), same trace: SPEC acceptance 8
mkdir -p gpurun_out/policy
python -m paper_2503_13737_b200.cli gen --out gpurun_out/policy/trace.jsonl --requests ${REQ:-400} --rate ${RATE:-8} \
  --long-fraction 0.1 --long-hi 16384 --profile profiles/opt13b_b200_tp1.json > gpurun_out/policy/gen.log 2>&1
timeout 1500 python -m paper_2503_13737_b200.cli run --trace gpurun_out/policy/trace.jsonl --profile profiles/opt13b_b200_tp1.json \
  --executor cuda --horizon ${HORIZON:-30} --kv-blocks ${KVB:-5300} \
  --policy accelgen --policy paged_fcfs --policy static_chunk --policy orca_fcfs \
  --out gpurun_out/policy > gpurun_out/policy/run.log 2>&1
python -m paper_2503_13737_b200.cli compare gpurun_out/policy/report_*.json --baseline paged_fcfs > gpurun_out/policy/compare.json 2>&1
