# K3 A/B: hybrid (CTG_K3_HYB=1) vs the default Montgomery Euclid, plus the GPU parity suite.  usage: bash scripts/ab_k3.sh [tag]
O=gpurun_out/${1:-hyb}; mkdir -p $O
CTG_K3_HYB=1 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest_exit=$? >> $O/pytest.log
Q="--no-cpu-baseline --no-headline"
for w in "d20_b64 256" "d30_b128 64" "d16_b1024 64"; do set -- $w
  CTG_K3_HYB=1 python bench.py --workload $1 --batch $2 $Q > $O/hyb_$1.json 2>$O/hyb_$1.err
  python bench.py --workload $1 --batch $2 $Q > $O/mont_$1.json 2>$O/mont_$1.err
done
tail -2 $O/pytest.log
for f in $O/*.json; do python -c "import json,sys;l=json.load(open('$f'));r=l['roofline'];print('$f',round(l['value']/1e9,3),round(l['e2e']['value']/1e9,3),round(r['frac'],3),{k:round(v,3) for k,v in r['stage_ms_per_step'].items()})"; done
