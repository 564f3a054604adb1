#!/bin/bash
# Measured side of the phase-B DRAM attribution (tools/l2_model_phase_b.py is the model): DRAM bytes of
# one phase-B launch (config 2 mini-sequence) for phase-B raster groups 4/8/16/32 and L2 policies.
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
for v in "MOM_GROUP_M_B=4" "MOM_GROUP_M_B=8" "MOM_GROUP_M_B=16" "MOM_GROUP_M_B=32" \
         "MOM_TMA_POLICY=1" "MOM_TMA_POLICY=5" "MOM_TMA_POLICY=2"; do
  echo "=== $v"
  env $v ncu --metrics $M --clock-control none --kernel-name-base demangled -k regex:"mlp_tc_kernel<.int.2, .int.1>" -s 1 -c 1 --csv python tools/one_minseq.py 2>&1 | grep -E "^\"" | tail -8
done
