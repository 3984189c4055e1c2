#!/bin/bash
# CRT carry kernel A/B: thread per coefficient vs warp per coefficient (CTG_CARRY_WARP_MAX).
# Measured on B200 (CRT stage ms, thread vs warp kernel): d20 B=256 0.229 vs 0.393; d30 B=64
# 0.336 vs 0.433; d16/1024 B=64 0.492 vs 0.634 -> warp kernel only for <= 4736 coefficients.
for w in "d20_b64 256" "d30_b128 64" "d16_b1024 64"; do set -- $w
  for mx in 0 100000000; do
    CTG_CARRY_WARP_MAX=$mx python bench.py --workload $1 --batch $2 --steps 5 --warmup 3 --no-cpu-baseline --no-headline 2>/dev/null > gpurun_out/abc.json
    python -c "
import json;d=json.load(open('gpurun_out/abc.json'));print('$1 B=$2 warp_max=$mx crt ms', round(d['roofline']['stage_ms_per_step']['crt'],4), 'step', round(d['ms_per_step'],3))"
  done
done
