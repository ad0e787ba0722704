#!/bin/bash
# Throughput of every mode on C2 and of EFT on every arc config, plus a size sweep (gpurun).
mkdir -p gpurun_out
OUT=gpurun_out/sweep.jsonl
: > $OUT
for m in eft eft_literal naive yac base naive_kahan; do
  python bench.py --mode $m --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline | tail -1 >> $OUT
done
for c in 3 5 6 7; do
  python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline | tail -1 >> $OUT
done
for n in 65536 1048576 4194304 67108864 268435456; do
  python bench.py --n $n --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline | tail -1 >> $OUT
done
echo sweep done
