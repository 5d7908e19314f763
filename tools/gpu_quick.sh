#!/bin/bash
# Quick GPU iteration: parity tests, phase traces, one bench line.  Usage: tools/gpu_quick.sh [bench args]
set -u
BARGS=("$@")
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
for cfg in "8 5 51865 f32 exact c2" "256 8 151936 f32 exact c4" "64 8 32000 f32 exact c3" "8 5 51865 f32 sigmoid c2"; do
  set -- $cfg
  timeout 60 python tools/trace_step.py --B $1 --gamma $2 --V $3 --dtype $4 --variant $5 > $OUT/trace_$6_$5.txt 2>&1
done
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu "${BARGS[@]}" > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
echo done
