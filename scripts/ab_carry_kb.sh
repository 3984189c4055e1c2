# CRT carry tile walk: limbs per load batch (CTG_CARRY_KB = 8, 16; 32 was measured with a
# temporary instantiation).  Result (B200, CRT stage ms): d16/1024 64 curves 0.498 / 0.461 / 0.558,
# d30/128 64 0.268 / 0.262 / 0.332, d20/64 256 0.205 / 0.205 / 0.250 -> default 16.
O=gpurun_out/${1:-kb}; mkdir -p $O
Q="--no-cpu-baseline --no-headline"
for w in "d16_b1024 64" "d30_b128 64" "d20_b64 256"; do set -- $w
  for kb in 8 16; do
    CTG_CARRY_KB=$kb python bench.py --workload $1 --batch $2 $Q > $O/kb${kb}_$1_$2.json 2>/dev/null
  done
done
for f in $O/*.json; do python -c "import json;l=json.load(open('$f'));s=l['roofline']['stage_ms_per_step'];print('$f','crt',round(s['crt'],4),'step',round(l['ms_per_step'],4))"; done
