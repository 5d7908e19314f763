#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
for i in 1 2; do python tools/sweep.py exact 1,5,32000,f32 8,5,51865,f32 64,8,32000,f32 64,8,32000,bf16 8,8,51865,bf16; done > $OUT/exp_sweep.txt 2>&1
echo done
