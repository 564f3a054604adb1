#!/bin/bash
# Round-end evidence on one B200: bench line (twice), launch list of a short bench run, ncu --set full of
# the last-token GEMVs (isolated tool), tests.  Outputs under gpurun_out/final/.
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_a.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/final/bench_b.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gate_up_gemv|down_gemv" -s 10 -c 2 \
    -o gpurun_out/final/gemv_full python tools/bench_gemv.py > gpurun_out/final/gemv_ncu.log 2>&1
ncu -i gpurun_out/final/gemv_full.ncu-rep --page raw --csv > gpurun_out/final/gemv_full_raw.csv 2>/dev/null
rm -f gpurun_out/final/gemv_full.ncu-rep
