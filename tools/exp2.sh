set -u
OUT=gpurun_out
SSV_RUNA=38 SSV_LAG_MULT=1000 timeout 120 python tools/trace_step.py --B 256 --gamma 8 --V 151936 > $OUT/trace_pm.txt 2>&1
SSV_RUNA=16 SSV_LAG_MULT=3 timeout 120 python tools/trace_step.py --B 256 --gamma 8 --V 151936 > $OUT/trace_r16m3.txt 2>&1
SSV_RUNA=38 SSV_LAG_MULT=1000 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_verify -s 3 -c 1 -o $OUT/ncu_pm -f python tools/prof_step.py --B 256 --gamma 8 --V 151936 --iters 5 > $OUT/ncu_pm.log 2>&1
