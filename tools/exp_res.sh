#!/bin/bash
# Cluster-path experiment: fold exponentials on the FMA pipe (SSV_DBG_MODE = npoly << 4), PDL off.
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="1,5,32000,f32 8,5,51865,f32 4,8,51865,f32 8,8,32000,f32 8,16,32000,f32 2,16,151936,f32 16,5,32000,f32 32,5,32000,f32 64,8,32000,f32 8,4,51865,f32"
for np in 0 1 2 3 4; do SSV_DBG_MODE=$((np*16)) timeout 300 python tools/sweep.py exact $SH > $OUT/poly_$np.txt 2>&1; done
SSV_NO_PDL=1 timeout 300 python tools/sweep.py exact $SH > $OUT/nopdl.txt 2>&1
SSV_DBG_MODE=48 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
SSV_DBG_MODE=48 timeout 60 python tools/trace_step.py --B 8 --gamma 5 --V 51865 --dtype f32 --variant exact > $OUT/trace_c2_on.txt 2>&1
