#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
FQ_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 --no-extras > gpurun_out/tp2.log 2>&1; echo "exit $?" >> gpurun_out/tp2.log
FQ_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 3 --warmup 3 --no-extras > gpurun_out/tp4.log 2>&1; echo "exit $?" >> gpurun_out/tp4.log
FQ_BENCH_ONE_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/tp2ref.log 2>&1; echo "exit $?" >> gpurun_out/tp2ref.log
