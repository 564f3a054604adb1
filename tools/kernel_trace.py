"""In-kernel timeline of the tcgen05 MLP launches in the bench's pipelined step (config 2):
%globaltimer stamps per CTA (entry, first MMA, last MMA, exit) via mom_set_kernel_trace.  Prints, per
launch, the MMA span and the gap from the previous launch's last MMA to this launch's first MMA, and
the share of the MLP wall time with no MMA being issued anywhere (transitions)."""
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
steps = int(os.environ.get("STEPS", "3"))
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
rows = []
for j in range(n):
    ent, fm, lm, ex, c0, c1 = (t[j, :, k] for k in range(6))
    used = ent > 0
    lead = fm > 0
    mhz = statistics.median(((c1[lead] - c0[lead]) / (lm[lead] - fm[lead]) * 1e3).tolist())
    ecyc, ecnt = t[j, :, 6], t[j, :, 7]
    epi = float(ecyc[used].sum() / max(1, ecnt[used].sum()))  # mean epilogue cycles per tile (warp 4)
    rows.append({"launch": j, "phase": "A" if j % 2 == 0 else "B", "ctas": int(used.sum()),
                 "entry_min": int(ent[used].min()), "entry_max": int(ent[used].max()),
                 "first_mma_min": int(fm[lead].min()), "first_mma_max": int(fm[lead].max()),
                 "last_mma_min": int(lm[lead].min()), "last_mma_max": int(lm[lead].max()), "exit_max": int(ex[used].max()),
                 "mhz": mhz, "epi_cycles": epi})
t0 = rows[0]["entry_min"]
gaps = []
for j, r in enumerate(rows):
    g = None if j == 0 else (r["first_mma_min"] - rows[j - 1]["last_mma_max"]) / 1e3
    if g is not None and not (j % (2 * wl.M) == 0):
        gaps.append((r["phase"], g))
    print(f'{j:3d} {r["phase"]} entry {(r["entry_min"]-t0)/1e3:9.1f}..{(r["entry_max"]-t0)/1e3:9.1f} '
          f'firstMMA {(r["first_mma_min"]-t0)/1e3:9.1f}..{(r["first_mma_max"]-t0)/1e3:9.1f} '
          f'lastMMA {(r["last_mma_min"]-t0)/1e3:9.1f}..{(r["last_mma_max"]-t0)/1e3:9.1f} exit {(r["exit_max"]-t0)/1e3:9.1f} us'
          + f' {r["mhz"]:6.0f} MHz epi {r["epi_cycles"]:7.0f} cyc' + ("" if g is None else f'  gap {g:7.1f}'))
ga = [g for p, g in gaps if p == "B"]   # A(i) -> B(i)
gb = [g for p, g in gaps if p == "A"]   # B(i) -> A(i+1)
per_step_us = (rows[-1]["exit_max"] - rows[0]["entry_min"]) / 1e3 / steps
mA = [r["mhz"] for r in rows if r["phase"] == "A"]
mB = [r["mhz"] for r in rows if r["phase"] == "B"]
eA = [r["epi_cycles"] for r in rows if r["phase"] == "A"]
eB = [r["epi_cycles"] for r in rows if r["phase"] == "B"]
print(json.dumps({"phaseA_mhz_median": round(statistics.median(mA)), "phaseB_mhz_median": round(statistics.median(mB)),
                  "phaseA_epilogue_cycles_per_tile": round(statistics.median(eA)),
                  "phaseB_epilogue_cycles_per_tile": round(statistics.median(eB))}))
print(json.dumps({"launches": n, "A_to_B_gap_us_mean": round(statistics.mean(ga), 2),
                  "B_to_A_gap_us_mean": round(statistics.mean(gb), 2) if gb else None,
                  "mlp_wall_us_per_step": round(per_step_us, 1),
                  "gap_share": round((sum(ga) + sum(gb)) / steps / per_step_us, 4)}))
