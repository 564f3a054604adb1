#!/bin/bash
# In-bench last-token GEMV pair: load-queue variant x head-of-row W_down L2 prefetch (KB per row) before
# the down GEMV waits for gate/up; gate_up PDL on.  2 interleaved rounds.
python -m pytest tests/test_gpu_knobs.py -x -q 2>&1 | tail -1
for r in 1 2; do for v in 1 2; do for pf in 0 4 12; do
  out=$(MOM_GEMV_VARIANT=$v MOM_GEMV_PREFETCH=$pf python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "round=$r variant=$v prefetch_kb=$pf $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(json.dumps({"step_ms": round(d["ms_per_step"],3), "gemv_us": round(k["last_token_gemv"]["ms"]*1e3,1), "gemv_frac": round(k["last_token_gemv"]["frac_hbm"],3), "head_us": round(k["lm_head_gemv"]["ms"]*1e3,1)}))')"
done; done; done
