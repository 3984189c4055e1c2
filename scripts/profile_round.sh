#!/bin/bash
# Round profile capture (run under gpurun): launch list of the default bench command and one
# ncu --set full capture per hot kernel at d30/128 (batch 4).  Plain runs first (exit 0 gate).
set -e
mkdir -p gpurun_out/prof
DEF="python bench.py --steps 2 --warmup 1 --batch 64 --no-cpu-baseline --no-headline"
$DEF > gpurun_out/prof/plain_default.json 2> gpurun_out/prof/plain_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
    --log-file gpurun_out/prof/launches_default.csv $DEF > gpurun_out/prof/ncu_default.log 2>&1
D30="python bench.py --workload d30_b128 --batch 4 --steps 1 --warmup 1 --no-cpu-baseline --no-headline"
$D30 > gpurun_out/prof/plain_d30.json 2> gpurun_out/prof/plain_d30.err
for k in k_modres_fast k_eval_ntt k_crt_gemm_i8 k_crt_carry8 k_interp k_reduce; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof/full_d30_$k $D30 \
      > gpurun_out/prof/ncu_d30_$k.log 2>&1 || true
done
