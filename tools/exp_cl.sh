#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
S=""
for V in 32000 51865 151936; do for g in 1 4 8 16; do for B in 1 4 16 32 64; do S="$S $B,$g,$V,f32"; done; done; done
timeout 900 python tools/sweep.py exact $S > $OUT/sw_cl.txt 2>&1
SSV_NO_CLUSTER=1 timeout 900 python tools/sweep.py exact $S > $OUT/sw_st.txt 2>&1
echo done
