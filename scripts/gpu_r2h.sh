#!/bin/bash
# re-entry check of HEAD: whole -m gpu suite + smoke + default bench line
TAG=r2h bash scripts/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/r2h_bench.jsonl 2> gpurun_out/r2h_bench.err
echo "bench rc=$?" >> gpurun_out/r2h_bench.err
tail -2 gpurun_out/r2h_bench.err
