#!/bin/bash
# Ring plan streaming pieces of the row slices (default rule vs SSV_PIECES=1).
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="64,8,32000,f32 64,8,32000,bf16 32,8,32000,f32 48,8,32000,f32 64,5,32000,f32 64,4,32000,f32 32,16,32000,f32 16,8,51865,f32 32,5,51865,f32 64,5,51865,f32 48,5,51865,f32 64,2,51865,f32 24,8,151936,bf16 16,4,151936,f32"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
SSV_PIECES=1 timeout 300 python tools/sweep.py exact $SH > $OUT/pc_1.txt 2>&1
SSV_DEBUG=1 timeout 300 python tools/sweep.py exact $SH > $OUT/pc_d.txt 2>&1
SSV_PIECES=1 timeout 300 python tools/sweep.py exact $SH > $OUT/pc_1b.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/pc_db.txt 2>&1
