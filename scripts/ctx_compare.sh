#!/bin/bash
# The reference's own caller CurveContext(f) (R = res(f, f_y) + Yun(R), lift.cpp:59-68) and its
# resultant_q()/q_factorization() (lift.cpp:76-101), built against the reference's elim.cpp
# (oracle/_ref/refdriver) and against the GPU drop-in TU (oracle/_ref/refdriver_gpu).
O=gpurun_out/ctx
mkdir -p $O
for c in "dense 10 10" "dense 12 10" "sheared 2 0" "sheared 3 0" "dense 16 64" "dense 20 64" "dense 30 128" "dense 16 1024"; do
  set -- $c
  timeout 120 oracle/_ref/refdriver_gpu time_ctx $1 $2 $3 1 5 q >> $O/gpu.jsonl 2>> $O/gpu.err
done
for c in "dense 10 10" "dense 12 10" "sheared 2 0" "sheared 3 0"; do
  set -- $c
  timeout 300 oracle/_ref/refdriver time_ctx $1 $2 $3 1 1 q >> $O/ref.jsonl 2>> $O/ref.err
done
