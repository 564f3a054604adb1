#!/bin/bash
# Phase-A raster group sizes near 16 (74 pairs: each A panel is shared by 74/G concurrent clusters).
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for g in 14 16 18 20; do
  env MOM_GROUP_M_A=$g ITERS=1 ROUNDS=1 timeout 300 ncu --metrics $M --clock-control none -k regex:mlp_tc_kernel -s 6 -c 1 --csv python tools/energy_sweep.py 2>/dev/null | grep -E "mlp_tc" | awk -v v="G=$g" -F'","' '{print v" | "$5" | "$(NF-2)" "$NF}'
done
ROUNDS=4 timeout 900 python tools/energy_sweep.py '{"MOM_GROUP_M_A":"16"}' '{"MOM_GROUP_M_A":"18"}' '{"MOM_GROUP_M_A":"14"}' '{"MOM_GROUP_M_A":"20"}'
