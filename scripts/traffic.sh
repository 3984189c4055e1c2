#!/bin/bash
# DRAM traffic of the K3 launch in the bench's own command (roofline "traffic"): plain run
# first (exit-0 gate), then ONE ncu --set full capture of the first k_modres_fast launch
# (a warm-up step of the same batch), then profiles/traffic.json via scripts/traffic_json.py.
# usage: scripts/traffic.sh <workload> [batch]
W=${1:-d20_b64}; B=${2:-64}
mkdir -p gpurun_out/traffic
CMD="python bench.py --workload $W --batch $B --steps 1 --warmup 3 --no-cpu-baseline --no-headline"
$CMD > gpurun_out/traffic/plain_$W.json 2> gpurun_out/traffic/plain_$W.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_modres_fast -c 1 \
    -o gpurun_out/traffic/k3_${W}_b$B $CMD > gpurun_out/traffic/ncu_$W.log 2>&1 || exit 1
python scripts/traffic_json.py $W $B gpurun_out/traffic/k3_${W}_b$B.ncu-rep
