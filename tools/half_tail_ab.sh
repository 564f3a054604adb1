python -m pytest tests/test_gpu_knobs.py tests/test_gpu_parity.py tests/test_gpu_random_shapes.py tests/test_gpu_edge.py tests/test_gpu_fused.py -x -q > gpurun_out/t_ht.log 2>&1
ROUNDS=4 python tools/energy_sweep.py '{"MOM_HALF_TAIL":"1"}' '{"MOM_HALF_TAIL":"0"}' > gpurun_out/ht_sweep.txt 2>&1
for i in 1 2; do
  echo "on  $(MOM_HALF_TAIL=1 python bench.py --no-cpu-baseline --no-e2e | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernels"]["phaseA_tc"]["ms"], d["clocks"]["sm_mhz"])')" >> gpurun_out/ht_bench.txt
  echo "off $(MOM_HALF_TAIL=0 python bench.py --no-cpu-baseline --no-e2e | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernels"]["phaseA_tc"]["ms"], d["clocks"]["sm_mhz"])')" >> gpurun_out/ht_bench.txt
done
