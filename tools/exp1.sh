set -u
OUT=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python tools/dbg_probs.py > $OUT/dbg.txt 2>&1
run() { # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --workload ${WL:-c4} --variant ${VAR:-exact} --steps ${ST:-200} --warmup 5 --no-cpu --no-extra > $OUT/exp_$name.json 2>$OUT/exp_$name.err
  python -c "
import json;d=json.load(open('$OUT/exp_$name.json'));print('$name', round(d['ms_per_step']*1e3,1),'us/step', round(d['roofline']['kernel_ms']*1e3,1),'us kernel', round(d['roofline']['frac'],3))" >> $OUT/exp_summary.txt 2>&1
}
ST=30 run c4_aonly_r2 SSV_AONLY=1 SSV_RUNA_FORCE=2
ST=30 run c4_aonly_r4 SSV_AONLY=1 SSV_RUNA_FORCE=4
ST=30 run c4 X=1
ST=30 WL=c4bf16 run c4bf16 X=1
WL=c3 run c3 X=1
WL=c3bf16 run c3bf16 X=1
