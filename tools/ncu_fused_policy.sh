#!/bin/bash
# DRAM bytes of the fused single launch vs the split path under L2 policies 0/1.
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for v in "MOM_FUSED=0 MOM_TMA_POLICY=0" "MOM_FUSED=0 MOM_TMA_POLICY=1" "MOM_FUSED=1 MOM_TMA_POLICY=0" "MOM_FUSED=1 MOM_TMA_POLICY=1" "MOM_FUSED=1 MOM_TMA_POLICY=1 MOM_GROUP_M_A=8"; do
  env $v ITERS=1 ROUNDS=1 ncu --metrics $M --clock-control none -k regex:mlp_tc_kernel -s 6 -c 2 --csv python tools/energy_sweep.py 2>/dev/null | grep -E "mlp_tc_kernel" | awk -v v="$v" -F'","' '{print v" | "$5" | "$(NF-2)" "$NF}'
done
