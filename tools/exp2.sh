set -u
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
for c in "8 5 51865" "1 5 32000"; do set -- $c
timeout 100 python tools/trace_step.py --B $1 --gamma $2 --V $3 >> $OUT/trace_cl.txt 2>&1
done
