#!/bin/bash
# Phase-A raster group size: DRAM bytes per launch (ncu) and the energy sweep (interleaved rounds).
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
for g in 16 24 32; do
  env MOM_GROUP_M_A=$g ITERS=1 ROUNDS=1 ncu --metrics $M --clock-control none -k regex:mlp_tc_kernel -s 6 -c 2 --csv python tools/energy_sweep.py 2>/dev/null | grep -E "mlp_tc_kernel" | awk -v v="MOM_GROUP_M_A=$g" -F'","' '{print v" | "$5" | "$(NF-2)" "$NF}'
done
ROUNDS=4 python tools/energy_sweep.py '{"MOM_GROUP_M_A":"16"}' '{"MOM_GROUP_M_A":"32"}' '{"MOM_GROUP_M_A":"24"}'
