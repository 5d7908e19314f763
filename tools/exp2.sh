set -u
OUT=gpurun_out
timeout 300 python tools/dbg_probs.py > $OUT/dbg.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
