#!/bin/bash
# Last-token GEMV pair inside the bench step (power-capped clock, after phase B): load-queue variants x
# PDL launch of gate_up; per-kernel event time from bench.py's event-timed pass, 2 interleaved rounds.
python -m pytest tests/test_gpu_knobs.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for r in 1 2; do for v in 1 2 3; do for pdl in 1 0; do
  out=$(MOM_GEMV_VARIANT=$v MOM_GEMV_PDL=$pdl python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "round=$r variant=$v pdl=$pdl $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(json.dumps({"step_ms": round(d["ms_per_step"],3), "gemv_us": round(k["last_token_gemv"]["ms"]*1e3,1), "gemv_frac": round(k["last_token_gemv"]["frac_hbm"],3), "head_us": round(k["lm_head_gemv"]["ms"]*1e3,1), "sm_mhz": d["clocks"]["sm_mhz"]}))')"
done; done; done
