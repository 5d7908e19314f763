#!/bin/bash
# Round profile: bench line, ncu launch list of the bench command, one ncu --set full per workload.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:k_verify -c 200 --csv --log-file $OUT/launches.csv python bench.py --steps 30 --warmup 3 --no-extra --no-cpu --no-e2e > $OUT/ncu_bench.out 2>&1
for cfg in "8 5 51865 f32 exact c2" "256 8 151936 f32 exact c4" "64 8 32000 f32 exact c3" "8 5 51865 f32 sigmoid c2" "256 8 151936 f32 sigmoid c4" "256 8 151936 bf16 exact c4bf16" "1 5 32000 f32 exact c1"; do
  set -- $cfg
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_verify -s 3 -c 1 \
     -o $OUT/ncu_$6_$5 -f python tools/prof_step.py --B $1 --gamma $2 --V $3 --dtype $4 --variant $5 --iters 5 > $OUT/ncu_$6_$5.log 2>&1
done
# summarise on the box (reports are large): markdown + json + per-line hot spots, keep two reports
python tools/ncu_summary.py $OUT/round_ncu.md $OUT/ncu_summary.json c2-exact=$OUT/ncu_c2_exact.ncu-rep \
   c3-exact=$OUT/ncu_c3_exact.ncu-rep c4-exact=$OUT/ncu_c4_exact.ncu-rep c2-sigmoid=$OUT/ncu_c2_sigmoid.ncu-rep \
   c4-sigmoid=$OUT/ncu_c4_sigmoid.ncu-rep c4bf16-exact=$OUT/ncu_c4bf16_exact.ncu-rep c1-exact=$OUT/ncu_c1_exact.ncu-rep > /dev/null 2>&1
for w in c2_exact c4_exact c4_sigmoid; do python tools/ncu_lines.py $OUT/ncu_$w.ncu-rep 25 > $OUT/lines_$w.txt 2>&1; done
python tools/ncu_launches.py $OUT/launches.csv > $OUT/launches.txt 2>&1
rm -f $OUT/ncu_c1_exact.ncu-rep $OUT/ncu_c3_exact.ncu-rep $OUT/ncu_c2_sigmoid.ncu-rep $OUT/ncu_c4_sigmoid.ncu-rep $OUT/ncu_c4bf16_exact.ncu-rep
du -sh $OUT
echo done
