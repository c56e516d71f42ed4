#!/bin/bash
# ncu evidence for the round-2 bench: (1) launch list of the timed windows, (2) --set full of the first
# attention / GEMM launches of the timed window, (3) TP=2 bench plumbing on one GPU (host collectives)
TAG=${TAG:-r2f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
mkdir -p gpurun_out/plan_cache
export AG_GEMM_PLAN_CACHE=gpurun_out/plan_cache
RAMP=${RAMP:-60}
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv env AG_NCU_TIMED=1 python bench.py --steps 2 --warmup 1 --ramp-s $RAMP \
  --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.out 2> gpurun_out/${TAG}_ncu_bench.err
echo "launch list rc=$?" >> gpurun_out/${TAG}_log.txt
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt 2>&1
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"mixed_attention|gemm" --launch-count ${NFULL:-12} -o gpurun_out/${TAG}_bench_full \
  env AG_NCU_TIMED=1 python bench.py --steps 1 --warmup 1 --ramp-s $RAMP --no-cpu-baseline --kv-gb ${NCU_KV_GB:-40} \
  > gpurun_out/${TAG}_full.out 2> gpurun_out/${TAG}_full.err
echo "full rc=$?" >> gpurun_out/${TAG}_log.txt
python scripts/ncu_summary.py gpurun_out/${TAG}_bench_full.ncu-rep > gpurun_out/${TAG}_full_summary.txt 2>&1
if [ -z "$SKIP_TP" ]; then
timeout 900 python bench.py --gpus 2 --tp-backend host --steps 3 --warmup 1 --ramp-s 20 --rate 1 --kv-gb 20 \
  > gpurun_out/${TAG}_tp2.out 2> gpurun_out/${TAG}_tp2.err
echo "tp2 rc=$?" >> gpurun_out/${TAG}_log.txt
fi
cat gpurun_out/${TAG}_log.txt; head -20 gpurun_out/${TAG}_launch_summary.txt; cat gpurun_out/${TAG}_full_summary.txt | head -20
