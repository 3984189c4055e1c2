#!/bin/bash
# Round-2 profile capture (one GPU, under gpurun).  Plain runs first (exit-0 gate), then
#   1. the launch list of the DEFAULT bench command (d30/128, 64 curves + the d20 extra),
#   2. one ncu --set full capture per hot kernel of the default workload (first launch each),
#   3. the Yun d30 launch list + one ncu --set full of k_modyun (the 3-prime probe),
#   4. K3 DRAM traffic of the default workload (profiles/traffic.json).
set -e
O=gpurun_out/prof_r02
mkdir -p $O
DEF="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-headline"
$DEF > $O/plain_default.json 2> $O/plain_default.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv $DEF > $O/ncu_default.log 2>&1
ONE="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-headline --no-extra"
for k in k_modres_fast k_eval_ntt k_gemm_u8_carry k_crt_fixup k_crt_prep_t k_interp k_reduce; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/full_$k $ONE > $O/ncu_full_$k.log 2>&1 || true
done
python scripts/yun_launches.py > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_yun_d30.csv python scripts/yun_launches.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_modyun -c 1 -o $O/full_k_modyun python scripts/yun_launches.py > $O/ncu_full_k_modyun.log 2>&1 || true
python scripts/traffic_json.py d30_b128 64 $O/full_k_modres_fast.ncu-rep > $O/traffic.log 2>&1 || true
cp profiles/traffic.json $O/traffic.json || true
echo profile_r02 done
