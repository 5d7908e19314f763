#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
S="1,5,32000,f32 8,5,51865,f32 64,8,32000,f32 64,8,32000,bf16 256,8,151936,f32 256,8,151936,bf16 32,8,151936,f32"
{
echo "== poly2 (default)"; python tools/sweep.py exact $S
echo "== poly1"; SSV_LIB=$PWD/build/libssv_poly1.so python tools/sweep.py exact $S
echo "== poly0"; SSV_LIB=$PWD/build/libssv_poly0.so python tools/sweep.py exact $S
} > $OUT/exp_sweep.txt 2>&1
echo done
