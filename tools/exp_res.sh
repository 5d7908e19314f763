#!/bin/bash
# A/B: paired granule loads in the cluster kernel (new build) vs tools/libssv_old.so.
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="64,8,32000,f32 64,8,32000,bf16 64,8,51865,bf16 64,5,51865,f32 32,8,51865,f32 48,8,32000,f32 8,5,51865,f32 8,5,51865,bf16 1,5,32000,f32 16,8,51865,f32 16,5,32000,bf16"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
SSV_LIB=tools/libssv_old.so timeout 300 python tools/sweep.py exact $SH > $OUT/a0.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/a1.txt 2>&1
SSV_LIB=tools/libssv_old.so timeout 300 python tools/sweep.py exact $SH > $OUT/a0b.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/a1b.txt 2>&1
