#!/bin/bash
# usage: scripts/launches.sh <workload> <tag> [batch]: plain run, then the ncu launch list
# (per-kernel device times, cold-cache and serialised: compare shares, not absolutes).
W=$1; T=$2; B=${3:-64}
mkdir -p gpurun_out/launches
CMD="python bench.py --workload $W --batch $B --steps 1 --warmup 3 --no-cpu-baseline --no-headline"
$CMD > gpurun_out/launches/plain_$T.json 2> gpurun_out/launches/plain_$T.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
    --log-file gpurun_out/launches/launches_$T.csv $CMD > gpurun_out/launches/ncu_$T.log 2>&1
