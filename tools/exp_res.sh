#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="64,8,32000,f32 64,8,32000,bf16 64,8,51865,bf16 48,8,51865,bf16 64,5,51865,bf16 64,5,51865,f32 48,5,51865,f32 32,8,51865,f32 64,8,51865,f32 32,8,51865,bf16 64,16,32000,f32 32,5,51865,f32 40,6,51865,f32"
SSV_PIECE_KB=12 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
timeout 300 python tools/sweep.py exact $SH > $OUT/k16.txt 2>&1
SSV_PIECE_KB=12 timeout 300 python tools/sweep.py exact $SH > $OUT/k12.txt 2>&1
SSV_PIECE_KB=10 timeout 300 python tools/sweep.py exact $SH > $OUT/k10.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/k16b.txt 2>&1
SSV_PIECE_KB=12 timeout 300 python tools/sweep.py exact $SH > $OUT/k12b.txt 2>&1
