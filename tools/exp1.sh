set -u
OUT=gpurun_out
run() { # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --workload ${WL:-c4} --variant ${VAR:-exact} --steps 200 --warmup 5 --no-cpu --no-extra > $OUT/exp_$name.json 2>$OUT/exp_$name.err
  python -c "
import json;d=json.load(open('$OUT/exp_$name.json'));print('$name', round(d['ms_per_step']*1e3,1),'us/step', round(d['roofline']['kernel_ms']*1e3,1),'us kernel', round(d['roofline']['frac'],3))" >> $OUT/exp_summary.txt 2>&1
}
for w in c1 c2 c3; do for v in exact sigmoid; do
WL=$w VAR=$v run ${w}_${v}_cluster X=1
WL=$w VAR=$v run ${w}_${v}_stream SSV_NO_CLUSTER=1
done; done
