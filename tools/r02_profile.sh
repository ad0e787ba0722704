#!/bin/bash
# Round-2 GPU measurement helper (run under gpurun from the repo root):
#   tools/r02_profile.sh <tag> [bench args for the ncu capture]
# 1. host facts; 2. FP64 microbenchmarks; 3. ncu launch list of a short default bench;
# 4. one ncu --set full capture of the EFT kernel on C2 and on C5 (2^30, traffic per launch).
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
{ free -g; nproc; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; } > $OUT/${TAG}_host.txt 2>&1
# the FP64 microbenchmarks (git-ignored binaries): build them if absent
[ -x tools/fp64_peak ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
[ -x tools/fp64_mix ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/fp64_mix tools/fp64_mix.cu
./tools/fp64_peak > $OUT/${TAG}_fp64_peak.json 2>&1
./tools/fp64_mix > $OUT/${TAG}_fp64_mix.txt 2>&1
ARGS="--steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-accuracy"
python bench.py $ARGS --config 2 > $OUT/${TAG}_plain_c2.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py $ARGS > $OUT/${TAG}_ncu_launches.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sgi_intersect_tma -s 3 -c 1 \
    -o $OUT/${TAG}_eft_c2 -f python bench.py $ARGS --config 2 > $OUT/${TAG}_eft_c2_ncu.log 2>&1
echo "full capture C2 rc=$?"
ncu --set full --clock-control none -k regex:sgi_intersect_tma -s 3 -c 1 \
    -o $OUT/${TAG}_eft_c5 -f python bench.py $ARGS > $OUT/${TAG}_eft_c5_ncu.log 2>&1
echo "full capture C5 rc=$?"
