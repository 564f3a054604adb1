#!/bin/bash
# Down GEMV K-split over 2 / 4 warps per row group (MOM_GEMV_VARIANT=5 / 6) vs the default (2): tests,
# isolated cold/hot (configs 2-4), inside the bench step, ncu durations of the down kernels.
timeout 600 python -m pytest tests/test_gpu_knobs.py -x -q -k "ksplit or bit_neutral" 2>&1 | tail -1
for r in 1 2; do for cfg in 1 2 3; do for v in 2 5 6; do for hot in 0 1; do
  echo "round=$r cfg=$cfg variant=$v hot=$hot $(MOM_GEMV_VARIANT=$v HOT=$hot CFG=$cfg timeout 300 python tools/bench_gemv.py)"
done; done; done; done
for r in 1 2; do for v in 2 5 6; do
  out=$(MOM_GEMV_VARIANT=$v timeout 600 python bench.py --no-stack --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "inbench round=$r variant=$v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(json.dumps({"step_ms": round(d["ms_per_step"],3), "gemv_us": round(k["last_token_gemv"]["ms"]*1e3,1), "gemv_frac": round(k["last_token_gemv"]["frac_hbm"],3)}))')"
done; done
for v in 2 5 6; do
  echo "ncu variant=$v $(MOM_GEMV_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"down_gemv" -c 3 --csv python tools/bench_gemv.py 2>&1 | grep -E '^"[0-9]' | awk -F'","' '{printf "%s ", $15}')"
done
