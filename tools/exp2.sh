set -u
OUT=gpurun_out
for m in 1 2; do
timeout 120 env SSV_LAG_MULT=$m python tools/trace_step.py --B 8 --gamma 5 --V 51865 > $OUT/trace_c2_m$m.txt 2>&1
timeout 120 env SSV_LAG_MULT=$m python tools/trace_step.py --B 64 --gamma 8 --V 32000 > $OUT/trace_c3_m$m.txt 2>&1
done
timeout 120 python tools/trace_step.py --B 8 --gamma 5 --V 51865 --variant sigmoid > $OUT/trace_c2_sig.txt 2>&1
