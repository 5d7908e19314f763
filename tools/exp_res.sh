#!/bin/bash
# A/B: all-resident one-CTA-per-SM cluster plan vs the two-per-SM ring plan.
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="1,5,32000,f32 8,5,51865,f32 8,5,51865,bf16 4,8,51865,f32 8,8,32000,f32 8,16,32000,f32 4,16,51865,f32 2,16,151936,f32 8,2,151936,f32 16,5,32000,f32 32,5,32000,f32 64,8,32000,f32 1,16,151936,f32 8,4,51865,f32 12,5,51865,f32 4,5,51865,f32"
for m in 1 2; do SSV_RES_MODE=$m SSV_DEBUG=1 timeout 300 python tools/sweep.py exact $SH > $OUT/res_$m.txt 2>&1; done
for cs in 16 11 10 9; do SSV_FORCE_CS=$cs SSV_DEBUG=1 timeout 300 python tools/sweep.py exact 8,5,51865,f32 8,5,51865,bf16 > $OUT/res_cs$cs.txt 2>&1; done
timeout 60 python tools/trace_step.py --B 8 --gamma 5 --V 51865 --dtype f32 --variant exact > $OUT/trace_c2_on.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 > $OUT/pytest_par.txt 2>&1; echo rc=$? >> $OUT/pytest_par.txt
