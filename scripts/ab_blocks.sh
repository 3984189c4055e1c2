#!/bin/bash
# e2e A/B of the batch block policy (CTG_BLOCK_MAX middle blocks, CTG_BLOCK_HEAD first/last)
# with two compute streams (superseded by scripts/ab_streams.sh, which also varies the stream
# count: the default is now 3 streams and 64-curve middle blocks).
for cfg in "128 32" "192 32" "96 32" "64 16" "128 16" "256 16"; do set -- $cfg
  export CTG_BLOCK_MAX=$1 CTG_BLOCK_HEAD=$2
  r=""
  for i in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-headline --steps 10 2>/dev/null > gpurun_out/blk.json
    r="$r $(python -c "import json;d=json.load(open('gpurun_out/blk.json'));print(round(d['e2e']['value']/1e9,3))")"
  done
  echo "max=$1 head=$2 e2e:$r"
done
