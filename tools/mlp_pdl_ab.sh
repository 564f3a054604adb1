#!/bin/bash
# Interleaved bench runs: tcgen05 MLP launches with / without PDL (MOM_MLP_PDL).
for i in 1 2 3; do
  for v in 0 1; do
    MOM_MLP_PDL=$v python bench.py --no-cpu-baseline | python -c "import json,sys; r=json.loads(sys.stdin.readlines()[-1]); print(json.dumps({'pdl': $v, 'ms': r['ms_per_step'], 'value': r['value'], 'phaseA_ms': r['kernels']['phaseA_tc']['ms'], 'phaseB_ms': r['kernels']['phaseB_tc']['ms'], 'e2e_ms': r['e2e']['ms_per_step'], 'serial_ms': r['serial']['ms_per_step'], 'sm_mhz': r['clocks']['sm_mhz']}))"
  done
done
