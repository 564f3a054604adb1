"""Where the bench step's time goes: launch-by-launch timeline (CUDA events recorded by the
library around each kernel) of a few pipelined config-2 steps, and the gaps between launches.
Usage: python tools/step_timeline.py [--serial]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2504_12526_b200 import _mom  # noqa: E402

serial = "--serial" in sys.argv

# copy-engine intervals: wrap the KV entries so each copy is bracketed by events on its stream
copies = []
_off, _rel = _mom.kv_offload, _mom.kv_reload


def _offload(kv, host, producer=None, copy=None, *a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    copy.wait_stream(producer)
    e0.record(copy)
    r = _off(kv, host, producer, copy, *a, **k)
    e1.record(copy)
    copies.append(("kv_offload D2H", e0, e1))
    return r


def _reload(host, kv, copy=None, *a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(copy)
    r = _rel(host, kv, copy, *a, **k)
    e1.record(copy)
    copies.append(("kv_reload H2D", e0, e1))
    return r


_mom.kv_offload, _mom.kv_reload = _offload, _reload
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
wl = bench.Workload(synth.CONFIGS[1], 0, 1, dev)
compute, copy, reload = (torch.cuda.Stream(dev) for _ in range(3))
with torch.cuda.stream(compute):
    for _ in range(5):
        bench.run_step(wl, compute, copy, reload, [0], serial=serial)
    bench.join_streams(compute, copy, reload)
torch.cuda.synchronize()
timer = _mom.LaunchTimer(capacity=256)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 4
copies.clear()
with timer, torch.cuda.stream(compute):
    ev0.record(compute)
    for _ in range(steps):
        bench.run_step(wl, compute, copy, reload, [0], serial=serial)
    bench.join_streams(compute, copy, reload)
    ev1.record(compute)
torch.cuda.synchronize()
tl = timer.timeline(ev0)
total = ev0.elapsed_time(ev1)
busy = sum(e - s for _, s, e in tl)
prev_end = 0.0
gaps = {}
for kind, s, e in tl:
    key = f"before {kind}"
    gaps.setdefault(key, []).append(s - prev_end)
    prev_end = e
print(f"{'serial' if serial else 'pipelined'}: {steps} steps {total:.3f} ms ({total / steps:.3f} ms/step), "
      f"kernels busy {busy:.3f} ms, idle {total - busy:.3f} ms, tail after last launch {total - prev_end:.3f} ms")
for k, v in gaps.items():
    print(f"  gap {k:28s} n={len(v):3d} mean {1e3 * sum(v) / len(v):8.1f} us  max {1e3 * max(v):8.1f} us")
for kind, s, e in tl[: 2 * wl.M + 3]:
    print(f"  {kind:18s} {s:9.3f} {e:9.3f}  ({1e3 * (e - s):8.1f} us)")
print("copy-engine intervals (ms from the origin; a copy's start waits for its stream's dependencies):")
for name, e0, e1 in copies:
    print(f"  {name:18s} {ev0.elapsed_time(e0):9.3f} {ev0.elapsed_time(e1):9.3f}  ({e0.elapsed_time(e1):7.3f} ms, "
          f"{wl.kv.numel() * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9:5.1f} GB/s)")
