#!/bin/bash
# DRAM bytes per tcgen05 MLP launch (config 2) in three contexts: an isolated mini-sequence with ncu's
# default cache flush, and the bench's pipelined step with the flush (all) and without it (none: the
# L2 state the previous launch left, as in the timed step).
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second"
out=gpurun_out/dram; mkdir -p $out
ncu --metrics $M --clock-control none -k regex:mlp_tc_kernel -s 2 -c 2 --csv python tools/one_minseq.py > $out/isolated_flush.csv 2>&1
for cc in all none; do
  ncu --metrics $M --clock-control none --cache-control $cc -k regex:mlp_tc_kernel -s 64 -c 8 --csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-stack > $out/bench_$cc.csv 2>&1
done
