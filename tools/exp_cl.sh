#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
python tools/sweep.py exact 1,5,32000,f32 8,5,51865,f32 64,8,32000,f32 64,8,32000,bf16 > $OUT/exp_sweep.txt 2>&1
timeout 60 python tools/trace_step.py --B 8 --gamma 5 --V 51865 > $OUT/trace_c2.txt 2>&1
echo done
