set -u
OUT=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
run() { # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --workload ${WL:-c4} --variant ${VAR:-exact} --steps ${ST:-200} --warmup 5 --no-cpu --no-extra > $OUT/exp_$name.json 2>$OUT/exp_$name.err
  python -c "
import json;d=json.load(open('$OUT/exp_$name.json'));print('$name', round(d['ms_per_step']*1e3,1),'us/step', round(d['roofline']['kernel_ms']*1e3,1),'us kernel', round(d['roofline']['frac'],3))" >> $OUT/exp_summary.txt 2>&1
}
ST=30 WL=c4bf16 run c4bf16 X=1
ST=30 WL=c4 run c4 X=1
WL=c3 run c3 X=1
ST=30 WL=c4 VAR=sigmoid run c4sig X=1
ST=30 WL=c4bf16 VAR=sigmoid run c4bf16sig X=1
