set -u
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
for c in "8 5 51865" "1 5 32000"; do set -- $c
SSV_DEBUG=1 timeout 100 python tools/trace_step.py --B $1 --gamma $2 --V $3 >> $OUT/trace_cl.txt 2>&1
done
cat > /tmp/x.sh <<'EOS'
EOS
for w in c1 c2; do for v in exact sigmoid; do
timeout 300 python bench.py --workload $w --variant $v --steps 300 --warmup 5 --no-cpu --no-extra > $OUT/b_${w}_$v.json 2>/dev/null
python -c "import json;d=json.load(open('$OUT/b_${w}_$v.json'));print('$w $v', round(d['ms_per_step']*1e3,2), 'us/step')" >> $OUT/exp_summary.txt
done; done
