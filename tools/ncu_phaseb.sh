#!/bin/bash
# DRAM bytes of phase A/B under raster/policy variants (one ncu --metrics pass per variant)
for v in "MOM_GROUP_M_B=8" "MOM_GROUP_M_B=2" "MOM_GROUP_M_B=1" "MOM_GROUP_M_B=1 MOM_TMA_POLICY=5" "MOM_GROUP_M_B=2 MOM_TMA_POLICY=5" "MOM_GROUP_M_B=32"; do
  env $v ITERS=1 ROUNDS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:mlp_tc_kernel -s 6 -c 2 --csv python tools/energy_sweep.py 2>/dev/null | grep -E "mlp_tc_kernel" | awk -v v="$v" -F'","' '{print v" | "$5" | "$(NF-2)" "$(NF-1)" "$NF}'
done
