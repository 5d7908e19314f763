set -u
OUT=gpurun_out
timeout 300 python tools/dbg_probs.py > $OUT/dbg.txt 2>&1
for tool in memcheck racecheck synccheck; do
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool python tools/dbg_probs.py > $OUT/san_$tool.txt 2>&1
done
