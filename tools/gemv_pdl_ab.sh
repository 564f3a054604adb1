#!/bin/bash
# Does the PDL launch of gate_up (behind the last phase B) cost the MLP anything?  Step time, in-kernel
# MMA-issue efficiency of the MLP step, GEMV time; MOM_GEMV_PDL=1 vs 0, 3 interleaved rounds.
for r in 1 2 3; do for pdl in 1 0; do
  out=$(MOM_GEMV_PDL=$pdl python bench.py --no-stack --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "round=$r pdl=$pdl $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; t=d["kernel_trace"]; print(json.dumps({"step_ms": round(d["ms_per_step"],3), "step_eff": t["mlp_step_mma_issue_efficiency"], "B_eff": t["phaseB_mma_issue_efficiency"], "mhz": t["phaseA_mhz"], "gemv_us": round(k["last_token_gemv"]["ms"]*1e3,1), "B_tflops": round(k["phaseB_tc"]["tflops"])}))')"
done; done
