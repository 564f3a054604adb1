#!/bin/bash
# Phase-A epilogue SiLU quotient: rcp.approx (MOM_FAST_SILU=1) vs IEEE division.  (The round-1 run also
# timed the since-removed wide-tile prototype, MOM_WIDE=1: profiles/r1_wide_tile_experiment.txt.)
timeout 600 python -m pytest tests/test_gpu_knobs.py tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_random_shapes.py -x -q > gpurun_out/fs_t.log 2>&1
echo "tests rc=$?" >> gpurun_out/fs_t.log
M="gpu__time_duration.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for v in "MOM_FAST_SILU=0" "MOM_FAST_SILU=1"; do
  env $v ITERS=1 ROUNDS=1 timeout 300 ncu --metrics $M --clock-control none -k regex:mlp_tc -s 6 -c 2 --csv python tools/energy_sweep.py 2>/dev/null | grep -E "mlp_tc" | awk -v v="$v" -F'","' '{print v" | "$5" | "$(NF-2)" "$NF}'
done > gpurun_out/fs_ncu.txt
ROUNDS=5 timeout 900 python tools/energy_sweep.py '{"MOM_FAST_SILU":"0"}' '{"MOM_FAST_SILU":"1"}' > gpurun_out/fs_sweep.txt 2>&1
