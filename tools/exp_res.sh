#!/bin/bash
# Resident slices copied as SSV_SPLIT bulk copies (folds start on the first chunks).
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="8,5,51865,f32 8,5,51865,bf16 1,5,32000,f32 1,5,32000,bf16 4,8,51865,f32 8,4,51865,f32 4,5,51865,f32 8,2,151936,f32 1,16,151936,f32"
SSV_SPLIT=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
for q in 1 2 4 8; do SSV_SPLIT=$q timeout 300 python tools/sweep.py exact $SH > $OUT/q$q.txt 2>&1; done
SSV_SPLIT=1 timeout 300 python tools/sweep.py exact $SH > $OUT/q1b.txt 2>&1
SSV_SPLIT=4 timeout 60 python tools/trace_step.py --B 8 --gamma 5 --V 51865 --dtype f32 --variant exact > $OUT/trace_c2.txt 2>&1
