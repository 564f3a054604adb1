#!/bin/bash
# Interleaved bench runs: cross-request reload overlap (default) vs --serial.
for i in 1 2; do
  for m in "" "--serial"; do
    python bench.py --no-cpu-baseline $m | python -c "import json,sys; r=json.loads(sys.stdin.readlines()[-1]); print(json.dumps({'mode': '$m' or 'pipelined', 'ms': r['ms_per_step'], 'value': r['value'], 'phaseA_tflops': r['kernels']['phaseA_tc']['tflops'], 'frac': r['roofline']['frac'], 'sm_mhz': r['clocks']['sm_mhz'], 'serial_ms': r.get('serial', {}).get('ms_per_step'), 'e2e_ms': r['e2e']['ms_per_step']}))"
  done
done
