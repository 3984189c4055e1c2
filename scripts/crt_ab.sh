#!/bin/bash
# A/B of the CRT stage: fused carry epilogue (default) vs CTG_CRT_UNFUSED=1, launch lists of
# the d20/256 and d30/64 bench workloads (kernel durations under ncu, cold caches).
O=gpurun_out/crt_ab; mkdir -p $O
for u in 0 1; do
  for w in "d20_b64 256" "d30_b128 64"; do set -- $w
    CTG_CRT_UNFUSED=$u ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_${1}_u$u.csv \
      python bench.py --workload $1 --batch $2 --steps 2 --warmup 1 --no-cpu-baseline --no-headline --no-extra > /dev/null 2>&1
  done
done
