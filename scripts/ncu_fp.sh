#!/bin/bash
# FP64-prime experiment: one ncu --set full of the fast mod-p kernel per CTG_FP_FRAC value.
mkdir -p gpurun_out/fpn
CMD="python bench.py --workload d20_b64 --batch 8 --steps 1 --warmup 1 --no-cpu-baseline --no-headline"
for f in 0 0.5 1.0; do
  CTG_FP_FRAC=$f $CMD > gpurun_out/fpn/plain_$f.json 2>&1 || exit 1
  CTG_FP_FRAC=$f ncu --set full --clock-control none --import-source on -k regex:k_modres_fast -c 1 -o gpurun_out/fpn/k3_$f $CMD > gpurun_out/fpn/ncu_$f.log 2>&1
done
