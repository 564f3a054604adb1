#!/bin/bash
# The N > 1 code paths on a one-GPU box (both ranks on cuda:0, gloo + host barriers; timings are not
# measurements): default bench (config 2 weak scaling, fused gather, e2e) and --stack (config 5 split,
# first 4 layers), plus smoke().
MOM_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 2>&1 | tail -2
MOM_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29542 bench.py --stack --layers 4 --gpus 2 --steps 2 --warmup 3 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
