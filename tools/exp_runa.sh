#!/bin/bash
# Experiment: A-run length at the streaming shapes (experiment build).
set -u
OUT=gpurun_out/runa
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
export SSV_LIB=$PWD/build/libssv_exp.so
for R in 0 8 4 2 1; do
  if [ $R -gt 0 ]; then export SSV_RUNA_FORCE=$R; else unset SSV_RUNA_FORCE; fi
  timeout 300 python tools/sweep.py --tag runa=$R --path streaming exact 256,8,151936,f32 256,8,151936,bf16 32,8,151936,f32 64,8,32000,f32 >> $OUT/sweep.txt 2>&1
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_verify -s 3 -c 1 \
     python tools/prof_step.py --B 256 --gamma 8 --V 151936 --iters 5 > $OUT/ncu_c4_runa$R.txt 2>&1
done
echo done
