set -u
OUT=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_verify -s 3 -c 1 -o $OUT/ncu_c1_cluster -f python tools/prof_step.py --B 1 --gamma 5 --V 32000 --iters 5 > $OUT/ncu_c1.log 2>&1
