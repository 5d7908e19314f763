set -u
OUT=gpurun_out
run() { # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --workload ${WL:-c4} --steps 20 --warmup 3 --no-cpu --no-extra > $OUT/exp_$name.json 2>$OUT/exp_$name.err
  python -c "
import json;d=json.load(open('$OUT/exp_$name.json'));print('$name', round(d['roofline']['kernel_ms']*1e3,1),'us', round(d['roofline']['frac'],3))" >> $OUT/exp_summary.txt 2>&1
}
for r in 12 16 24 38; do for m in 2 3 4 6; do run c4_r${r}_m$m SSV_RUNA=$r SSV_LAG_MULT=$m; done; done
WL=c3; for r in 2 4 8; do for m in 1 2 3; do run c3_r${r}_m$m SSV_RUNA=$r SSV_LAG_MULT=$m; done; done
WL=c3bf16; for r in 4 8; do for m in 1 2 3; do run c3b_r${r}_m$m SSV_RUNA=$r SSV_LAG_MULT=$m; done; done
WL=c2; for r in 1 2; do for m in 1 2; do run c2_r${r}_m$m SSV_RUNA=$r SSV_LAG_MULT=$m; done; done
