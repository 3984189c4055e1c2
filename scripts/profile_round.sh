#!/bin/bash
# Round profile capture (run under gpurun, one GPU): plain runs first (exit-0 gate), then
#   1. the launch list of the DEFAULT bench command (ncu --metrics gpu__time_duration.sum),
#   2. K3 DRAM traffic at the default batch (profiles/traffic.json, copied to gpurun_out/prof),
#   3. one ncu --set full capture per hot kernel of the default workload (first launch each).
# usage: scripts/profile_round.sh [tag]
set -e
T=${1:-r01}
O=gpurun_out/prof_$T
mkdir -p $O
DEF="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-headline"
$DEF > $O/plain_default.json 2> $O/plain_default.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_default.csv $DEF > $O/ncu_default.log 2>&1
B=$(python -c "import json;print(json.load(open('$O/plain_default.json'))['config']['curves_per_step'])")
ONE="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-headline"
for k in k_modres_fast k_eval_ntt k_gemm_u8_tma k_crt_carry k_crt_prep_t k_interp k_reduce; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/full_$k $ONE \
      > $O/ncu_full_$k.log 2>&1 || true
done
python scripts/traffic_json.py d20_b64 $B $O/full_k_modres_fast.ncu-rep > $O/traffic.log 2>&1 || true
cp profiles/traffic.json $O/traffic.json || true
