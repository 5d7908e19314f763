#!/bin/bash
# Resident 16-warp plan: rows 8-9 split between two warps (default) vs whole rows (SSV_DBG_MODE=16).
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="8,5,51865,f32 8,5,51865,bf16 1,5,32000,f32 1,5,32000,bf16 4,5,51865,f32 8,5,32000,f32 2,5,151936,f32 6,5,51865,f32"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
SSV_DBG_MODE=16 timeout 300 python tools/sweep.py exact $SH > $OUT/x0.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/x1.txt 2>&1
SSV_DBG_MODE=16 timeout 300 python tools/sweep.py exact $SH > $OUT/x0b.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/x1b.txt 2>&1
timeout 60 python tools/trace_step.py --B 8 --gamma 5 --V 51865 --dtype f32 --variant exact > $OUT/trace_c2.txt 2>&1
