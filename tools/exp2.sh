set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
SSV_NO_PDL=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu > $OUT/bench_nopdl.json 2> $OUT/bench_nopdl.err
