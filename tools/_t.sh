mkdir -p gpurun_out/full
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/full/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/full/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/full/smoke.txt
timeout 900 python bench.py > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err; echo "bench rc=$?" >> gpurun_out/full/bench.err
