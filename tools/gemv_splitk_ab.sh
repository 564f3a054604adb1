#!/bin/bash
# Last-token MLP: two-launch GEMV pair (MOM_GEMV_VARIANT=1) vs the split-K single-stream kernel (2),
# isolated (cold: L2 flushed; hot: right after an MLP call), configs 2-4 shapes, interleaved x3;
# then one ncu pass over the split-K kernels.
for r in 1 2 3; do
  for cfg in 1 2 3; do
    for v in 1 2; do
      for hot in 0 1; do
        echo "round=$r cfg=$cfg variant=$v hot=$hot $(MOM_GEMV_VARIANT=$v HOT=$hot CFG=$cfg python tools/bench_gemv.py)"
      done
    done
  done
done
