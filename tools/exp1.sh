set -u
OUT=gpurun_out
mkdir -p $OUT
rm -f $OUT/exp_summary.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
run() { # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --workload ${WL:-c4} --variant ${VAR:-exact} --steps ${ST:-100} --warmup 5 --no-cpu --no-extra > $OUT/exp_$name.json 2>$OUT/exp_$name.err
  python -c "
import json;d=json.load(open('$OUT/exp_$name.json'));print('$name', round(d['ms_per_step']*1e3,1),'us/step', round(d['roofline']['kernel_ms']*1e3,1),'us kernel', round(d['roofline']['frac'],3))" >> $OUT/exp_summary.txt 2>&1
}
for i in 1 2; do
run c4_tail$i X=1
run c4_notail$i SSV_NO_TAIL=1
WL=c4bf16 run c4bf16_tail$i X=1
WL=c4bf16 run c4bf16_notail$i SSV_NO_TAIL=1
WL=c3 run c3_tail$i X=1
WL=c3 run c3_notail$i SSV_NO_TAIL=1
done
for cfg in "256 8 151936 f32 exact c4"; do
  set -- $cfg
  timeout 60 python tools/trace_step.py --B $1 --gamma $2 --V $3 --dtype $4 --variant $5 > $OUT/trace_$6_$5.txt 2>&1
  SSV_NO_TAIL=1 timeout 60 python tools/trace_step.py --B $1 --gamma $2 --V $3 --dtype $4 --variant $5 > $OUT/trace_$6_$5_notail.txt 2>&1
done
echo done
