#!/bin/bash
# Round-2 closing evidence on one B200 (outputs under gpurun_out/final_r2/): GPU suite, smoke, the default
# bench line twice, the reference arm, the ncu launch list of a short bench run, and one ncu --set full
# capture of phase A inside the bench step (bench's `traffic` field) -- all from the same tree.
out=gpurun_out/final_r2; mkdir -p $out
python -m pytest tests -m gpu -q -rA > $out/gputest.log 2>&1; tail -1 $out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
python bench.py > $out/bench_a.json 2> $out/bench_a.err
python bench.py --no-cpu-baseline > $out/bench_b.json 2> $out/bench_b.err
python bench.py --impl reference > $out/reference.json 2> $out/reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-stack > $out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled -k regex:"mlp_tc_kernel<.int.2, .int.0>" -s 40 -c 1 \
    -o $out/phaseA_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-stack > $out/phaseA_ncu.log 2>&1
ncu -i $out/phaseA_full.ncu-rep --page raw --csv > $out/phaseA_full_raw.csv 2>/dev/null
ncu -i $out/phaseA_full.ncu-rep --page details > $out/phaseA_full_details.txt 2>/dev/null
rm -f $out/phaseA_full.ncu-rep
