#!/bin/bash
# LM-head GEMV variants (MOM_HEAD_VARIANT, a temporary knob since removed: 0 = 4 rows x 2 loads, 1 = 2 rows x 4 loads per lane), cold and hot.
for i in 1 2; do for v in 0 1; do for h in 0 1; do
  echo "variant=$v hot=$h $(MOM_HEAD_VARIANT=$v HOT=$h python tools/bench_gemv.py)"
done; done; done
