#!/bin/bash
# Bench A/B: request i's last-token tail on its own stream (overlapping request i+1's MLP; default) vs on
# the compute stream (--no-tail-overlap).  3 interleaved rounds, config 2, default K/W.
python -m pytest tests/test_gpu_bench_pipeline.py -x -q 2>&1 | tail -1
for r in 1 2 3; do for v in "" "--no-tail-overlap"; do
  out=$(python bench.py --no-cpu-baseline $v 2>/dev/null | tail -1)
  echo "round=$r [$v] $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d.get("energy",{}); print(json.dumps({"value": round(d["value"]), "step_ms": round(d["ms_per_step"],3), "e2e": round(d["e2e"]["value"]), "serial_ms": round(d["serial"]["ms_per_step"],3), "J_step": round(e.get("joules_per_step",0),3), "mhz": d["clocks"]["sm_mhz"], "gemv_us": round(d["kernels"]["last_token_gemv"]["ms"]*1e3,1), "head_us": round(d["kernels"]["lm_head_gemv"]["ms"]*1e3,1)}))')"
done; done
