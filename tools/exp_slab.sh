#!/bin/bash
# Experiment: slab kernel vs streaming / cluster at the large exact shapes.
set -u
OUT=gpurun_out/slab
mkdir -p $OUT
SH="256,8,151936,f32 256,8,151936,bf16 32,8,151936,f32 64,8,32000,f32 64,8,32000,bf16 32,8,51865,f32"
timeout 300 python tools/sweep.py --tag slab --path slab exact 256,8,151936,f32 > $OUT/first.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "slab or c4_every or campaign" > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
for P in slab auto; do
  timeout 300 python tools/sweep.py --tag $P --path $P exact $SH >> $OUT/sweep.txt 2>&1
done
export SSV_LIB=$PWD/build/libssv_exp.so
for D in 1 3 4; do
  SSV_SLAB_DP=$D timeout 300 python tools/sweep.py --tag dp$D --path slab exact $SH >> $OUT/sweep.txt 2>&1
done
unset SSV_LIB
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_verify -s 3 -c 1 \
     python tools/prof_step.py --B 256 --gamma 8 --V 151936 --iters 5 > $OUT/ncu_c4.txt 2>&1
echo done
