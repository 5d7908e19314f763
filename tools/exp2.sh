set -u
OUT=gpurun_out
for c in "8 5 51865" "1 5 32000"; do set -- $c
timeout 100 python tools/trace_step.py --B $1 --gamma $2 --V $3 >> $OUT/trace_cl.txt 2>&1
done
timeout 100 python tools/trace_step.py --B 64 --gamma 8 --V 32000 >> $OUT/trace_cl.txt 2>&1
timeout 300 python tools/dbg_probs.py > $OUT/dbg.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
