#!/bin/bash
# Bench A/B (config 2 step, energy per step from the >= 2 s metered pass) of the epilogue L2 hints
# and the phase-A raster group, 2 interleaved rounds.
for r in 1 2; do for v in "MOM_EPI_L2_HINT=0 MOM_GROUP_M_A=16" "MOM_EPI_L2_HINT=1 MOM_GROUP_M_A=16" \
                          "MOM_EPI_L2_HINT=1 MOM_GROUP_M_A=32" "MOM_EPI_L2_HINT=3 MOM_GROUP_M_A=16" \
                          "MOM_EPI_L2_HINT=3 MOM_GROUP_M_A=32"; do
  out=$(env $v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "round=$r [$v] $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d.get("energy",{}); print(json.dumps({"step_ms": round(d["ms_per_step"],3), "A_tflops": round(d["kernels"]["phaseA_tc"]["tflops"]), "B_tflops": round(d["kernels"]["phaseB_tc"]["tflops"]), "J_step": round(e.get("joules_per_step",0),3), "e_step_ms": round(e.get("ms_per_step",0),3), "e_mhz": e.get("sm_mhz"), "mhz": d["clocks"]["sm_mhz"]}))')"
done; done
