#!/bin/bash
# A/B of library variants in _ab/*.so on the three bench workloads (stage times).
mkdir -p gpurun_out/ab
for lib in _ab/*.so; do for w in ${WORKLOADS:-d20_b64 d30_b128 d16_b1024}; do
  t=$(basename $lib .so)
  CTG_LIBRARY=$PWD/$lib python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-headline > gpurun_out/ab/${t}_$w.json 2> gpurun_out/ab/${t}_$w.err
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab/${t}_$w.json') if l.startswith('{')][-1]
print('$t','$w',round(d['ms_per_step'],3),'frac',round(d['roofline']['frac'],3),'e2e_ms/curve',round(d['e2e']['res_ms_per_curve'],4),{k:round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()})
"
done; done
