# Batch e2e block schedule A/B with priority chunk streams (d20, 256 curves), two runs each.
# Result (B200, 2 runs each, e2e 1e9 units/s): 32|64 3.85 3.83 (default) ; 16|64 3.71 3.67 ; 16|48 3.75 3.81 ; 32|96 3.48 3.39 ; 24|80 3.48 3.50
O=gpurun_out/${1:-blk}; mkdir -p $O
Q="--workload d20_b64 --batch 256 --no-cpu-baseline --no-headline --steps 20"
for rep in 1 2; do
for cfg in "32 64" "16 64" "16 48" "32 96" "24 80"; do set -- $cfg
  CTG_BLOCK_HEAD=$1 CTG_BLOCK_MAX=$2 python bench.py $Q > $O/h$1_m$2_$rep.json 2>/dev/null
done; done
for f in $O/*.json; do python -c "import json;l=json.load(open('$f'));print('$f','e2e',round(l['e2e']['value']/1e9,3),'ms/curve',round(l['e2e']['res_ms_per_curve']*1e3,2))"; done
