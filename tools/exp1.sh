set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 120 -k "host or optional" > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
python tools/e2e_probe.py > $OUT/e2e.txt 2>&1
timeout 300 python bench.py --steps 300 --warmup 5 --no-extra --no-cpu > $OUT/b.json 2>$OUT/b.err
python -c "import json;d=json.load(open('$OUT/b.json'));print(d['value'], d['e2e'])" > $OUT/exp_summary.txt 2>&1
