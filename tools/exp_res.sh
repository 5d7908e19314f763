#!/bin/bash
# Cluster-path experiment: parity, a shape sweep (with / without the bonus-row prefetch), the C2 phase trace.
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="1,5,32000,f32 8,5,51865,f32 8,5,51865,bf16 4,8,51865,f32 8,8,32000,f32 8,16,32000,f32 2,16,151936,f32 8,2,151936,f32 16,5,32000,f32 32,5,32000,f32 64,8,32000,f32 64,8,32000,bf16 8,4,51865,f32 4,5,51865,f32"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
timeout 300 python tools/sweep.py exact $SH > $OUT/res_2.txt 2>&1
SSV_DBG_MODE=4 timeout 300 python tools/sweep.py exact $SH > $OUT/res_nopf.txt 2>&1
timeout 300 python tools/sweep.py sigmoid $SH > $OUT/sig_2.txt 2>&1
SSV_DBG_MODE=4 timeout 300 python tools/sweep.py sigmoid $SH > $OUT/sig_nopf.txt 2>&1
timeout 60 python tools/trace_step.py --B 8 --gamma 5 --V 51865 --dtype f32 --variant exact > $OUT/trace_c2_on.txt 2>&1
