#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="64,5,51865,f32 48,5,51865,f32 32,5,51865,f32 64,8,51865,f32 32,8,51865,f32 64,8,51865,bf16 48,8,51865,f32 40,6,51865,f32 32,8,151936,f32 16,8,151936,f32 64,8,32000,f32 16,4,151936,f32 32,12,32000,f32 64,12,32000,f32"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
SSV_NO_CLUSTER=1 timeout 300 python tools/sweep.py exact $SH > $OUT/g0.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/g1.txt 2>&1
SSV_NO_GATE=1 timeout 300 python tools/sweep.py exact $SH > $OUT/g2.txt 2>&1
