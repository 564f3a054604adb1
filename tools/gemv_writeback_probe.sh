#!/bin/bash
# Does the last-token GEMV pay for phase B's dirty L2 lines?  ncu with --cache-control none (the real L2
# state at each launch) on the bench step: DRAM read / write bytes of the GEMV pair, with the phase-B
# output stores plain (MOM_EPI_L2_HINT=0) or evict_first (2); then the in-bench GEMV time A/B.
out=gpurun_out/wb; mkdir -p $out
for h in 0 2; do
  MOM_EPI_L2_HINT=$h ncu --cache-control none --clock-control none -k regex:"gate_up_gemv|down_gemv|lm_head_gemv" -s 30 -c 9 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $out/ncu_hint$h.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-stack > $out/ncu_hint$h.log 2>&1
done
for r in 1 2 3; do for h in 0 2; do
  echo "round=$r hint=$h $(MOM_EPI_L2_HINT=$h python bench.py --no-cpu-baseline --no-stack 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernels"]["last_token_gemv"]["ms"], d["kernels"]["lm_head_gemv"]["ms"], d["kernels"]["phaseB_tc"]["ms"], d["clocks"]["sm_mhz"])')"
done; done > $out/inbench.txt 2>&1
