#!/bin/bash
# A/B of the last-token GEMV pair's (rows per warp step, loads in flight, blocks per SM) variants,
# interleaved rounds, cold (L2 flushed) and hot (right after an MLP call).
for round in 1 2; do
  for v in 0 1 2 3 4 5 6; do
    echo "variant=$v round=$round cold $(MOM_GEMV_VARIANT=$v python tools/bench_gemv.py)"
    echo "variant=$v round=$round hot  $(MOM_GEMV_VARIANT=$v HOT=1 python tools/bench_gemv.py)"
  done
done
