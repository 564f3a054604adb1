"""Does the per-launch event timing inflate the bench step?  Pipelined config-2 steps with and
without the LaunchTimer, interleaved; and, without the timer, MLP launches with / without PDL."""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
import bench, synth
from paper_2504_12526_b200 import _mom
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
wl = bench.Workload(synth.CONFIGS[1], 0, 1, dev)
compute, copy, reload = (torch.cuda.Stream(dev) for _ in range(3))
def run(n, timed):
    timer = _mom.LaunchTimer(capacity=1024) if timed else None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if timer: timer.__enter__()
    with torch.cuda.stream(compute):
        e0.record(compute)
        for _ in range(n):
            bench.run_step(wl, compute, copy, reload, [0])
        bench.flush_reload(wl, reload)
        bench.join_streams(compute, copy, reload)
        e1.record(compute)
    if timer: timer.__exit__(None, None, None)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
run(5, False)
res = {}
for r in range(4):
    for name, t, pdl in (("no timer, pdl", False, "1"), ("timer, pdl", True, "1"), ("no timer, no pdl", False, "0"),
                         ("timer, no pdl", True, "0")):
        os.environ["MOM_MLP_PDL"] = pdl
        res.setdefault(name, []).append(run(20, t))
for name, v in res.items():
    print(f"{name:18s}", [round(x, 3) for x in v], round(statistics.mean(v), 3))
