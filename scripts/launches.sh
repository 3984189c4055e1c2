#!/bin/bash
# usage: scripts_launches.sh <workload> <tag>: plain run, then ncu launch list (per-kernel device times)
W=$1; T=$2
CMD="python bench.py --workload $W --batch 2 --steps 1 --warmup 1 --no-cpu-baseline --no-headline"
$CMD > gpurun_out/plain_$T.json 2> gpurun_out/plain_$T.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/launches_$T.csv $CMD > gpurun_out/ncu_$T.log 2>&1
