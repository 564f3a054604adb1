#!/bin/bash
# Down GEMV fed by bulk copies (MOM_GEMV_VARIANT=4) vs the register-fed default (2): tests, isolated
# (cold / hot, configs 2-4) and inside the bench step; ncu of both down kernels.
timeout 600 python -m pytest tests/test_gpu_knobs.py -x -q 2>&1 | tail -2
for r in 1 2; do for cfg in 1 2 3; do for v in 2 4; do for hot in 0 1; do
  echo "round=$r cfg=$cfg variant=$v hot=$hot $(MOM_GEMV_VARIANT=$v HOT=$hot CFG=$cfg timeout 300 python tools/bench_gemv.py)"
done; done; done; done
for r in 1 2; do for v in 2 4; do
  out=$(MOM_GEMV_VARIANT=$v timeout 600 python bench.py --no-stack --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "inbench round=$r variant=$v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(json.dumps({"step_ms": round(d["ms_per_step"],3), "gemv_us": round(k["last_token_gemv"]["ms"]*1e3,1), "gemv_frac": round(k["last_token_gemv"]["frac_hbm"],3)}))')"
done; done
MOM_GEMV_VARIANT=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gemv" -c 4 --csv python tools/bench_gemv.py 2>&1 | grep -E '^"[0-9]' | awk -F'","' '{print $5, $13, $15}'
