set -u
OUT=gpurun_out
run() { # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --workload ${WL:-c4} --steps 20 --warmup 3 --no-cpu --no-extra > $OUT/exp_$name.json 2>$OUT/exp_$name.err
  python -c "
import json;d=json.load(open('$OUT/exp_$name.json'));print('$name', round(d['roofline']['kernel_ms']*1e3,1),'us', round(d['roofline']['frac'],3))" >> $OUT/exp_summary.txt 2>&1
}
for r in 4 8 16 38; do run pm_r$r SSV_RUNA=$r SSV_LAG_MULT=1000; done
for r in 8 16; do run full_r${r}_m3 SSV_RUNA=$r SSV_LAG_MULT=3; done
WL=c3; for r in 1 2 4 8; do run c3_pm_r${r} SSV_RUNA=$r SSV_LAG_MULT=1000; done
WL=c3bf16; for r in 2 4 8; do run c3b_pm_r${r} SSV_RUNA=$r SSV_LAG_MULT=1000; done
WL=c2; for r in 1 2; do run c2_pm_r${r} SSV_RUNA=$r SSV_LAG_MULT=1000; done
