#!/bin/bash
# A/B of the fused K2+K3 kernel against the two-kernel path (default; CTG_FUSE=1 selects the fused kernel) on the bench
# workloads (stage times per step).  usage: scripts/ab_fuse.sh [batch]
B=${1:-64}
mkdir -p gpurun_out/abf
for w in ${WORKLOADS:-d20_b64 d30_b128 d16_b1024}; do for mode in fused split; do
  if [ $mode = fused ]; then export CTG_FUSE=1; else unset CTG_FUSE; fi
  python bench.py --workload $w --batch $B --steps 5 --warmup 3 --no-cpu-baseline --no-headline \
      > gpurun_out/abf/${mode}_$w.json 2> gpurun_out/abf/${mode}_$w.err
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/abf/${mode}_$w.json') if l.startswith('{')][-1]
print('$mode','$w',round(d['ms_per_step'],3),'frac',round(d['roofline']['frac'],3),'stage2',round(d['roofline']['stage2_frac'],3),'e2e_ms/curve',round(d['e2e']['res_ms_per_curve'],4),{k:round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()})
" || tail -5 gpurun_out/abf/${mode}_$w.err
done; done
unset CTG_FUSE
