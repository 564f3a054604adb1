#!/bin/bash
# r2 batch 2: GEMV load-queue variants (bit-neutral) A/B, LM head vs concurrent copies, phase-B DRAM
# attribution (ncu), configs 3/4 stacks (final-layer offload deferred after the head), knob tests.
python -m pytest tests/test_gpu_knobs.py tests/test_gpu_reload_pipelined.py tests/test_gpu_stack.py -x -q 2>&1 | tail -3 > gpurun_out/r2_b2_tests.log
for r in 1 2; do for cfg in 1 2 3; do for v in 1 2 3; do for hot in 0 1; do
  echo "round=$r cfg=$cfg variant=$v hot=$hot $(MOM_GEMV_VARIANT=$v HOT=$hot CFG=$cfg python tools/bench_gemv.py)"
done; done; done; done > gpurun_out/r2_gemv_queue_ab.txt 2>&1
python tools/head_copy_interference.py > gpurun_out/r2_head_copy_interference.json 2>&1
bash tools/ncu_phaseb_attribution.sh > gpurun_out/r2_phaseb_attribution.txt 2>&1
for c in 2 3; do timeout 900 python tools/bench_stack.py --config $c --steps 2 --warmup 1 >> gpurun_out/r2_stack_cfgs34_b.jsonl 2>> gpurun_out/r2_stack_cfgs34_b.err; done
