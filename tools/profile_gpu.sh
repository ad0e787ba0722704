#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run under gpurun from the repo root:
#   1. plain bench run (must exit 0), 2. ncu launch list (gpu__time_duration per launch),
#   3. one ncu --set full capture of the EFT kernel and of the naive kernel.
# Usage: tools/profile_gpu.sh <tag>
set -u
TAG=${1:-prof}
OUT=gpurun_out
mkdir -p $OUT
ARGS="--steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
python bench.py $ARGS > $OUT/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py $ARGS > $OUT/${TAG}_ncu_launches.log 2>&1
echo "launch list rc=$?"
for MODE in eft naive; do
  python bench.py --mode $MODE --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/${TAG}_${MODE}_plain2.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:sgi_intersect -s 4 -c 1 \
      -o $OUT/${TAG}_${MODE} python bench.py --mode $MODE --steps 3 --warmup 3 --e2e-steps 0 \
      --no-cpu-baseline > $OUT/${TAG}_${MODE}_ncu.log 2>&1
  echo "full capture $MODE rc=$?"
done
