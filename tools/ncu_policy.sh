#!/bin/bash
# DRAM bytes of the split path's phase A / phase B under the TMA L2-policy variants.
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
for v in "MOM_TMA_POLICY=0" "MOM_TMA_POLICY=1" "MOM_TMA_POLICY=3" "MOM_TMA_POLICY=4" "MOM_TMA_POLICY=1 MOM_GROUP_M_B=4" "MOM_TMA_POLICY=1 MOM_GROUP_M_B=16"; do
  env $v ITERS=1 ROUNDS=1 ncu --metrics $M --clock-control none -k regex:mlp_tc_kernel -s 6 -c 2 --csv python tools/energy_sweep.py 2>/dev/null | grep -E "mlp_tc_kernel" | awk -v v="$v" -F'","' '{print v" | "$5" | "$(NF-2)" "$NF}'
done
