#!/bin/bash
# usage: scripts/ncu_full.sh <workload> <batch> <tag> <kernel-regex>...   (plain run first, then one ncu --set full per kernel)
W=$1; B=$2; T=$3; shift 3
CMD="python bench.py --workload $W --batch $B --steps 1 --warmup 1 --no-cpu-baseline --no-headline"
$CMD > gpurun_out/plain_$T.json 2> gpurun_out/plain_$T.err || exit 1
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_${T}_$k $CMD > gpurun_out/ncu_${T}_$k.log 2>&1
done
