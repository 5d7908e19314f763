#!/bin/bash
# Resident plan also for slices that fit two CTAs per SM (padded to one per SM: SSV_RES_PAD).
set -u
OUT=gpurun_out; mkdir -p $OUT
SH="1,5,32000,f32 1,5,32000,bf16 1,2,32000,f32 2,5,32000,f32 4,5,32000,f32 8,5,32000,f32 8,8,32000,f32 8,5,51865,bf16 4,4,51865,f32 8,2,51865,f32 8,1,151936,f32 16,2,32000,f32 12,4,32000,f32 1,8,51865,f32 4,16,32000,bf16"
timeout 300 python tools/sweep.py exact $SH > $OUT/p0.txt 2>&1
SSV_RES_PAD=1 SSV_DEBUG=1 timeout 300 python tools/sweep.py exact $SH > $OUT/p1.txt 2>&1
timeout 300 python tools/sweep.py exact $SH > $OUT/p0b.txt 2>&1
