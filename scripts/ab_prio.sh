# Batch e2e A/B: chunk streams of decreasing priority (default) vs equal-priority rotation
# (CTG_CHUNK_PRIO=0); each arm run twice, interleaved.  usage: bash scripts/ab_prio.sh [tag]
O=gpurun_out/${1:-prio}; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest_exit=$? >> $O/pytest.log
Q="--no-cpu-baseline --no-headline"
for rep in 1 2; do
for w in "d20_b64 256" "d30_b128 64" "d16_b1024 64"; do set -- $w
  python bench.py --workload $1 --batch $2 $Q > $O/prio_$1_$rep.json 2>$O/prio_$1.err
  CTG_CHUNK_PRIO=0 python bench.py --workload $1 --batch $2 $Q > $O/rot_$1_$rep.json 2>$O/rot_$1.err
done; done
python scripts/trace_host.py "dense 20 64" 256 > $O/trace_prio.log 2>&1
tail -2 $O/pytest.log
for f in $O/*.json; do python -c "import json,sys;l=json.load(open('$f'));print('$f','value',round(l['value']/1e9,3),'e2e',round(l['e2e']['value']/1e9,3),l['e2e']['phases_ms_last_call'])"; done
tail -8 $O/trace_prio.log
