"""Probe build only (MOM_NVCC_EXTRA=-DMOM_TRACE_WAITS): where the MMA issuer of each tcgen05 MLP launch
waits, in the bench's pipelined config-2 step.  Per launch and leader CTA: cycles from its first to its
last MMA issue, cycles waiting for a full smem stage (operands late), cycles waiting for a free TMEM
accumulator (epilogue late), and the issue cycles the tiles need (128 per 256x256x16 pair MMA)."""
import ctypes, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import synth
from paper_2504_12526_b200 import _mom

dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
wl = bench.Workload(synth.CONFIGS[1], 0, 1, dev)
compute, copy, reload = (torch.cuda.Stream(dev) for _ in range(3))
with torch.cuda.stream(compute):
    for _ in range(3):
        bench.run_step(wl, compute, copy, reload, [0])
    bench.join_streams(compute, copy, reload)
torch.cuda.synchronize()
steps = 2
cap = steps * 2 * wl.M + 4
buf = torch.zeros(cap * 160 * 8, dtype=torch.int64, device=dev)
count = ctypes.c_int64(0)
_mom._check(_mom.lib().mom_set_kernel_trace(ctypes.c_void_p(buf.data_ptr()), cap, ctypes.byref(count)))
with torch.cuda.stream(compute):
    for _ in range(steps):
        bench.run_step(wl, compute, copy, reload, [0])
    bench.join_streams(compute, copy, reload)
torch.cuda.synchronize()
_mom.lib().mom_set_kernel_trace(None, 0, None)
n = count.value
t = buf.view(cap, 160, 8)[:n].cpu().numpy().astype("int64")
out = {"A": [], "B": []}
for j in range(n):
    ph = "A" if j % 2 == 0 else "B"
    fm, c0, c1, wf, wa = t[j, :, 1], t[j, :, 4], t[j, :, 5], t[j, :, 6], t[j, :, 7]
    lead = fm > 0
    span = (c1[lead] - c0[lead]).astype(float)
    out[ph].append({"span_cyc_med": float(statistics.median(span)), "wait_full_frac_med": float(statistics.median(wf[lead] / span)),
                    "wait_full_frac_max": float((wf[lead] / span).max()), "wait_acc_frac_med": float(statistics.median(wa[lead] / span)),
                    "wait_acc_frac_max": float((wa[lead] / span).max())})
for ph, rows in out.items():
    print(ph, json.dumps({k: round(statistics.median([r[k] for r in rows]), 4) for k in rows[0]}))
    for r in rows[:4]:
        print("   ", json.dumps({k: round(v, 4) for k, v in r.items()}))
