#!/bin/bash
# Phase-B column-group raster (MOM_RASTER_B_COLS): knob test, ncu DRAM bytes of one phase-B launch, and
# a bench A/B (step time + J/step from the metered >= 2 s pass), 3 interleaved rounds.
timeout 600 python -m pytest tests/test_gpu_knobs.py -x -q -k bit_neutral 2>&1 | tail -1
M=dram__bytes_read.sum,gpu__time_duration.sum
for v in "MOM_RASTER_B_COLS=0" "MOM_RASTER_B_COLS=4" "MOM_RASTER_B_COLS=8"; do
  echo "=== $v $(env $v ncu --metrics $M --clock-control none --kernel-name-base demangled -k regex:"mlp_tc_kernel<.int.2, .int.1>" -s 1 -c 1 --csv python tools/one_minseq.py 2>&1 | grep -E '^"[0-9]' | awk -F'","' '{printf "%s=%s ", $13, $15}')"
done
for r in 1 2 3; do for v in "MOM_RASTER_B_COLS=0" "MOM_RASTER_B_COLS=8"; do
  out=$(env $v timeout 600 python bench.py --no-stack --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "round=$r [$v] $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d.get("energy",{}); print(json.dumps({"step_ms": round(d["ms_per_step"],3), "B_tflops": round(d["kernels"]["phaseB_tc"]["tflops"]), "J_step": round(e.get("joules_per_step",0),3), "e_step_ms": round(e.get("ms_per_step",0),3), "mhz": e.get("sm_mhz")}))')"
done; done
