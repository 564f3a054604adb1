#!/bin/bash
# Companion captures to final_capture_r2.sh: ncu --set full of one phase-B launch and of the last-token GEMV
# pair + LM head inside the bench step (--cache-control none: the L2 state the step leaves), final code.
out=gpurun_out/final_r2b; mkdir -p $out
ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled \
    -k regex:"mlp_tc_kernel<.int.2, .int.1>" -s 40 -c 1 -o $out/phaseB_full \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-stack > $out/phaseB_ncu.log 2>&1
ncu -i $out/phaseB_full.ncu-rep --page raw --csv > $out/phaseB_full_raw.csv 2>/dev/null
ncu --set full --clock-control none --cache-control none --import-source on \
    -k regex:"gate_up_gemv|down_gemv|lm_head_gemv" -s 12 -c 3 -o $out/gemv_full \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-stack > $out/gemv_ncu.log 2>&1
ncu -i $out/gemv_full.ncu-rep --page raw --csv > $out/gemv_full_raw.csv 2>/dev/null
rm -f $out/*.ncu-rep
