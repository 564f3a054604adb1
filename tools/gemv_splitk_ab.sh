#!/bin/bash
# Last-token MLP: two-launch GEMV pair (MOM_GEMV_VARIANT=1) vs the split-K single-stream kernel (2; with
# 64-wide chunks = ceil(I/64) blocks, or MOM_SPLITK_BLOCKS_PER_SM=2), isolated (cold: L2 flushed; hot:
# right after an MLP call), config 2-4 shapes, interleaved x3.
for r in 1 2 3; do
  for cfg in 1 2 3; do
    for v in "MOM_GEMV_VARIANT=1" "MOM_GEMV_VARIANT=2" "MOM_GEMV_VARIANT=2 MOM_SPLITK_BLOCKS_PER_SM=2"; do
      for hot in 0 1; do
        echo "round=$r cfg=$cfg variant=[$v] hot=$hot $(env $v HOT=$hot CFG=$cfg python tools/bench_gemv.py)"
      done
    done
  done
done
