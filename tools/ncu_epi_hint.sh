#!/bin/bash
# DRAM bytes of one config-2 phase-A and phase-B launch for the epilogue L2 hints (MOM_EPI_L2_HINT:
# bit 0 H stores evict_first, bit 1 phase-B residual/out evict_first) x phase-A raster groups.
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum
for v in "MOM_EPI_L2_HINT=0 MOM_GROUP_M_A=16" "MOM_EPI_L2_HINT=1 MOM_GROUP_M_A=16" "MOM_EPI_L2_HINT=1 MOM_GROUP_M_A=24" \
         "MOM_EPI_L2_HINT=1 MOM_GROUP_M_A=32" "MOM_EPI_L2_HINT=0 MOM_GROUP_M_A=32" "MOM_EPI_L2_HINT=3 MOM_GROUP_M_A=16"; do
  echo "=== $v"
  env $v ncu --metrics $M --clock-control none --kernel-name-base demangled -k regex:"mlp_tc_kernel" -s 2 -c 2 --csv python tools/one_minseq.py 2>&1 | grep -E '^"[0-9]' | awk -F'","' '{print $5, $13, $15}'
done
