#!/bin/bash
# Token-sharded stack checks on a one-GPU box: the 2-process GPU test, bench.py --stack at N=1 and
# in the shared-GPU N=2 test mode (gloo + host barriers, timings meaningless), host memory info.
set -x
free -g
nvidia-smi --query-gpu=name,memory.total --format=csv
timeout 600 python -m pytest tests/test_gpu_stack_sharded.py -x -q -rA 2>&1 | tail -15
timeout 600 python bench.py --stack --layers 4 --steps 2 --warmup 3 2>&1 | tail -3
MOM_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --stack --layers 4 --gpus 2 --steps 2 --warmup 3 2>&1 | tail -5
