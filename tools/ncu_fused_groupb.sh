#!/bin/bash
# DRAM bytes of the fused single launch with phase-B sub-groups (MOM_GROUP_M_B) vs the split path.
# (Experiment script: the fused phase-B sub-group variant it measured was reverted; see profiles/r1_summary.md.)
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for v in "MOM_FUSED=0" "MOM_FUSED=1 MOM_GROUP_M_B=16" "MOM_FUSED=1" "MOM_FUSED=1 MOM_GROUP_M_B=4" "MOM_FUSED=1 MOM_GROUP_M_B=2"; do
  env $v ITERS=1 ROUNDS=1 ncu --metrics $M --clock-control none -k regex:mlp_tc_kernel -s 6 -c 2 --csv python tools/energy_sweep.py 2>/dev/null | grep -E "mlp_tc_kernel" | awk -v v="$v" -F'","' '{print v" | "$5" | "$(NF-2)" "$NF}'
done
