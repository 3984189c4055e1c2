#!/bin/bash
# e2e A/B of the number of compute streams the batch chunks rotate over (CTG_CHUNK_STREAMS)
# and of the largest middle block (CTG_BLOCK_MAX), d20 / 256 curves, 5 runs each.
# Measured (1e9 units/s): 2 streams / 128: 2.97-3.00; 2 / 64: 3.03-3.17; 3 / 128: 2.72-2.87;
# 3 / 64 (3 slots): 3.17-3.53 -> default 3 streams, 64-curve middle blocks, 4 slots.
for cfg in "${@:-3 64}"; do set -- $cfg
  r=""
  for i in 1 2 3 4 5; do
    CTG_CHUNK_STREAMS=$1 CTG_BLOCK_MAX=$2 python bench.py --no-cpu-baseline --no-headline --steps 10 2>/dev/null > gpurun_out/abs.json
    r="$r $(python -c "import json;d=json.load(open('gpurun_out/abs.json'));print(round(d['e2e']['value']/1e9,3))")"
  done
  echo "streams=$1 max=$2 e2e:$r"
done
