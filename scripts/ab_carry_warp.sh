# CRT carry A/B: warp per coefficient for every batch (CTG_CARRY_WARP_MAX large) vs the default
# threshold (tile walk above 4736 coefficients).  usage: bash scripts/ab_carry_warp.sh [tag]
# Result (B200, CRT stage ms tile / warp): d16/1024 64 curves 0.499 / 0.622, 16 curves 0.198 / 0.202;
# d30 64 0.269 / 0.398, 16 0.102 / 0.115; d20 256 0.205 / 0.360 -> threshold kept.
O=gpurun_out/${1:-cw}; mkdir -p $O
Q="--no-cpu-baseline --no-headline"
for w in "d16_b1024 64" "d30_b128 64" "d20_b64 256" "d16_b1024 16" "d30_b128 16"; do set -- $w
  python bench.py --workload $1 --batch $2 $Q > $O/tile_$1_$2.json 2>/dev/null
  CTG_CARRY_WARP_MAX=10000000 python bench.py --workload $1 --batch $2 $Q > $O/warp_$1_$2.json 2>/dev/null
done
for f in $O/*.json; do python -c "import json;l=json.load(open('$f'));s=l['roofline']['stage_ms_per_step'];print('$f','crt',round(s['crt'],4),'step',round(l['ms_per_step'],4),'e2e',round(l['e2e']['value']/1e9,3))"; done
