mkdir -p gpurun_out/fp
python -m pytest tests -m gpu -x -q > gpurun_out/fp/pytest.log 2>&1; tail -3 gpurun_out/fp/pytest.log
for f in 0 0.3 0.5 0.7 1.0; do for w in d20_b64 d30_b128 d16_b1024; do
CTG_FP_FRAC=$f python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-headline > gpurun_out/fp/b_${w}_$f.json 2> gpurun_out/fp/b_${w}_$f.err
python -c "
import json,sys
d=[json.loads(l) for l in open('gpurun_out/fp/b_${w}_$f.json') if l.startswith('{')][-1]
print('$f','$w',d['config']['primes'],round(d['ms_per_step'],3),round(d['value']/1e9,3),round(d['roofline']['frac'],3),{k:round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()})
"
done; done
