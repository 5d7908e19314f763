#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
python tools/sweep.py sigmoid 256,8,151936,f32 256,8,151936,bf16 128,8,51865,f32 1024,4,32000,f32 8,5,51865,f32 > $OUT/exp_sweep.txt 2>&1
echo done
SSV_LIB=$PWD/build/libssv_base.so python tools/sweep.py sigmoid 256,8,151936,f32 256,8,151936,bf16 128,8,51865,f32 1024,4,32000,f32 8,5,51865,f32 > $OUT/exp_sweep_base.txt 2>&1
