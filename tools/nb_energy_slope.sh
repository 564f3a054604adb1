#!/bin/bash
# Energy slope of L2->SM operand traffic from a natural tile-shape change: phase B with UMMA N = 256
# vs 128 (operand bytes per FLOP x1.5).  ncu lts/dram bytes per phase-B launch, then the interleaved
# energy sweep (whole 8-mini-sequence calls).
M="gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
for nb in 256 128; do
  env MOM_NB_B=$nb ITERS=1 ROUNDS=1 ncu --metrics $M --clock-control none -k regex:mlp_tc_kernel -s 6 -c 2 --csv python tools/energy_sweep.py 2>/dev/null | grep -E "mlp_tc_kernel" | awk -v v="MOM_NB_B=$nb" -F'","' '{print v" | "$5" | "$(NF-2)" "$NF}'
done
ROUNDS=5 python tools/energy_sweep.py '{"MOM_NB_B":"256"}' '{"MOM_NB_B":"128"}'
