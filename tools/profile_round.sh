#!/bin/bash
# Round profile: bench line, ncu launch list of the bench command, one ncu --set full per workload.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:k_verify -c 200 --csv --log-file $OUT/launches.csv python bench.py --steps 30 --warmup 3 --no-extra --no-cpu > $OUT/ncu_bench.out 2>&1
for cfg in "8 5 51865 f32 exact c2" "256 8 151936 f32 exact c4" "64 8 32000 f32 exact c3" "8 5 51865 f32 sigmoid c2" "256 8 151936 f32 sigmoid c4"; do
  set -- $cfg
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_verify -s 3 -c 1 \
     -o $OUT/ncu_$6_$5 -f python tools/prof_step.py --B $1 --gamma $2 --V $3 --dtype $4 --variant $5 --iters 5 > $OUT/ncu_$6_$5.log 2>&1
done
echo done
