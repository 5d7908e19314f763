#!/bin/bash
# One GPU session: tests, smoke, bench, launch list.  Usage: tools/gpu_check.sh [quick]
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | head -20 >> $OUT/nproc.txt
make -s -f paper_2406_11016_b200/csrc/Makefile > $OUT/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 180 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 --csv --log-file $OUT/launches.csv python bench.py --steps 30 --warmup 3 --no-extra --no-cpu > $OUT/ncu_bench.out 2>&1
echo done
