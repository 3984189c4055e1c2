#!/bin/bash
# The numbers DESIGN.md quotes (run under gpurun, one GPU): the default bench line, the
# other two headline workloads at 64 curves per step, and the Yun timings.
O=gpurun_out/numbers
mkdir -p $O
python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in d30_b128 d16_b1024 d10_b10; do
  python bench.py --workload $w --batch 64 --no-cpu-baseline --no-headline > $O/bench_$w.json 2> $O/bench_$w.err
done
python scripts/bench_yun.py > $O/yun.jsonl 2> $O/yun.err
