mkdir -p gpurun_out/sig
timeout 300 python tools/sweep.py --tag w5 sigmoid 1024,8,151936,f32 256,8,151936,f32 256,8,151936,bf16 256,8,32000,f32 512,8,51865,f32 > gpurun_out/sig/sweep14.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "c4_every or slab or sigmoid or eps or memory or determinism" > gpurun_out/sig/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/sig/pytest_gpu.txt
export SSV_LIB=$PWD/build/libssv_exp.so SSV_SLAB_TRACE=1 SSV_SIG_TRACE=1
timeout 120 python tools/trace_step.py --B 256 --gamma 8 --V 151936 --variant sigmoid > gpurun_out/sig/trace_c4.txt 2>&1
