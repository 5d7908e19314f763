set -u
OUT=gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 3 --no-extra --no-cpu --workload c4shard > $OUT/torchrun.json 2> $OUT/torchrun.err; echo "rc=$?" >> $OUT/torchrun.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $OUT/torchrun_ref.json 2> $OUT/torchrun_ref.err; echo "rc=$?" >> $OUT/torchrun_ref.err
