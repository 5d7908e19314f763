set -u
OUT=gpurun_out
run() { # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --workload ${WL:-c4} --variant ${VAR:-exact} --steps ${ST:-30} --warmup 5 --no-cpu --no-extra > $OUT/exp_$name.json 2>$OUT/exp_$name.err
  python -c "
import json;d=json.load(open('$OUT/exp_$name.json'));print('$name', round(d['ms_per_step']*1e3,1),'us/step', round(d['roofline']['kernel_ms']*1e3,1),'us kernel', round(d['roofline']['frac'],3))" >> $OUT/exp_summary.txt 2>&1
}
for r in 2 4 8 16; do run aonly_r$r SSV_AONLY=1 SSV_RUNA_FORCE=$r; done
for r in 4 8 16; do for m in 1 2 3; do run full_r${r}_m$m SSV_RUNA_FORCE=$r SSV_LAG_MULT=$m; done; done
