# Batch e2e block schedule for big outputs (d30/128, d16/1024: ~0.9 MB of limbs per curve),
# Result (B200, e2e 1e9 units/s, m = 64 / 32 / 16 / 8): d16/1024 64 curves 3.05 / 3.82 / 4.21 / 4.09, 256 curves 4.59 / 4.33 / 4.17 / 4.27;
# d30/128 64 curves 2.01 / 2.34 / 2.35 / 2.36, 256 curves 2.46 / 2.30 / 2.28 / 2.29 -> default: at least three middle blocks, <= 64.
# priority chunk streams: CTG_BLOCK_MAX (middle block) sweep, 64 and 256 curves.
O=gpurun_out/${1:-blkbig}; mkdir -p $O
for w in d16_b1024 d30_b128; do for B in 64 256; do for m in 64 32 16 8; do
  CTG_BLOCK_MAX=$m python bench.py --workload $w --batch $B --no-cpu-baseline --no-headline --steps 5 > $O/${w}_B${B}_m$m.json 2>/dev/null
done; done; done
for f in $O/*.json; do python -c "import json;l=json.load(open('$f'));print('$f','e2e',round(l['e2e']['value']/1e9,3),'val',round(l['value']/1e9,3))"; done
