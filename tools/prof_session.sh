#!/bin/bash
# Profiling session: phase traces + one ncu --set full capture per workload.
set -u
OUT=gpurun_out
mkdir -p $OUT
for cfg in "8 5 51865 f32 exact c2" "256 8 151936 f32 exact c4" "64 8 32000 f32 exact c3"; do
  set -- $cfg
  timeout 120 python tools/trace_step.py --B $1 --gamma $2 --V $3 --dtype $4 --variant $5 > $OUT/trace_$6_$5.txt 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_verify -s 3 -c 1 \
     -o $OUT/ncu_$6_$5 -f python tools/prof_step.py --B $1 --gamma $2 --V $3 --dtype $4 --variant $5 --iters 5 > $OUT/ncu_$6_$5.log 2>&1
done
echo done
