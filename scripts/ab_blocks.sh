#!/bin/bash
# e2e A/B of the batch block policy (CTG_BLOCK_MAX middle blocks, CTG_BLOCK_HEAD first/last).
# Measured on B200 (d20, 256 curves, e2e 1e9 units/s): 128/32 3.0-3.1 (default), 96/32 3.0,
# 64/16 3.0, 128/16 2.75, 192/32 2.6, 256/16 2.4.
for cfg in "128 32" "192 32" "96 32" "64 16" "128 16" "256 16"; do set -- $cfg
  export CTG_BLOCK_MAX=$1 CTG_BLOCK_HEAD=$2
  r=""
  for i in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-headline --steps 10 2>/dev/null > gpurun_out/blk.json
    r="$r $(python -c "import json;d=json.load(open('gpurun_out/blk.json'));print(round(d['e2e']['value']/1e9,3))")"
  done
  echo "max=$1 head=$2 e2e:$r"
done
