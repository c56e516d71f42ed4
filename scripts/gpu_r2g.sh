#!/bin/bash
# refined-policy rate sweep (2 s windows) then the ncu evidence + TP=2 plumbing
TAG=r2g RATES="3 4 5" BENCH_ARGS="--window-s 2" bash scripts/gpu_rate_sweep.sh
TAG=r2f bash scripts/gpu_r2_evidence.sh
