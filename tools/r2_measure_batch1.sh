#!/bin/bash
# r2 batch: phase-B DRAM attribution (ncu), TLB warm probe, config-5 stack at N=1 (32 layers, early vs
# Alg. 1 reload order), configs 3/4 stacks with both reload schedules.
bash tools/ncu_phaseb_attribution.sh > gpurun_out/r2_phaseb_attribution.txt 2>&1
for cfg in 2 3; do CFG=$cfg python tools/tlb_warm_probe.py >> gpurun_out/r2_tlb_probe.jsonl 2>&1; done
timeout 900 python bench.py --stack --steps 3 --warmup 3 > gpurun_out/r2_stack_cfg5_n1.json 2> gpurun_out/r2_stack_cfg5_n1.err
for c in 2 3; do timeout 900 python tools/bench_stack.py --config $c --steps 2 --warmup 1 >> gpurun_out/r2_stack_cfgs34.jsonl 2>> gpurun_out/r2_stack_cfgs34.err; done
