#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
SSV_DEBUG=1 timeout 60 python tools/trace_step.py --B 64 --gamma 8 --V 32000 --dtype f32 --variant exact > $OUT/trace_c3.txt 2>&1
timeout 60 python tools/trace_step.py --B 32 --gamma 5 --V 32000 --dtype f32 --variant exact > $OUT/trace_b32.txt 2>&1
