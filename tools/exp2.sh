set -u
OUT=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
for m in 0 2; do echo "== dbg $m" >> $OUT/trace_cl.txt
SSV_DBG_MODE=$m timeout 100 python tools/trace_step.py --B 1 --gamma 5 --V 32000 >> $OUT/trace_cl.txt 2>&1
done
timeout 100 python tools/trace_step.py --B 8 --gamma 5 --V 51865 >> $OUT/trace_cl.txt 2>&1
