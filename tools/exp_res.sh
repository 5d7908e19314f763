#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="1,5,32000,f32 1,5,32000,bf16 8,5,51865,f32 8,5,51865,bf16 8,8,32000,f32 4,8,51865,f32 16,5,32000,f32 32,5,32000,f32 64,8,32000,f32 64,8,32000,bf16 8,16,32000,f32 1,16,151936,f32"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
timeout 300 python tools/sweep.py exact $SH > $OUT/s1.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/s2.txt 2>&1
timeout 60 python tools/trace_step.py --B 8 --gamma 5 --V 51865 --dtype f32 --variant exact > $OUT/trace_c2.txt 2>&1
