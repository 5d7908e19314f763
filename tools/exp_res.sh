#!/bin/bash
# One-CTA-per-SM big-ring cluster plan (SSV_RING1) vs the default plans.
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="64,8,32000,f32 64,8,32000,bf16 32,8,32000,f32 48,8,32000,f32 64,5,32000,f32 64,4,32000,f32 32,16,32000,f32 16,8,51865,f32 64,8,51865,f32 16,8,151936,f32 32,5,51865,f32 16,16,32000,f32"
timeout 300 python tools/sweep.py exact $SH > $OUT/r1_0.txt 2>&1
SSV_RING1=1 SSV_DEBUG=1 timeout 300 python tools/sweep.py exact $SH > $OUT/r1_1.txt 2>&1
SSV_RING1=1 SSV_FORCE_CS=2 timeout 300 python tools/sweep.py exact $SH > $OUT/r1_cs2.txt 2>&1
SSV_RING1=1 timeout 60 python tools/trace_step.py --B 64 --gamma 8 --V 32000 --dtype f32 --variant exact > $OUT/trace_c3.txt 2>&1
