"""Energy-aware A/B of tcgen05 kernel variants at config 2 shapes.  On a power-capped B200
the clock follows energy per FLOP, so each variant reports TFLOP/s, mean SM clock, joules per
MLP call (NVML total-energy counter), TFLOP/J and TFLOP/s per GHz (per-cycle efficiency).
Variants are interleaved over rounds to cancel thermal drift.
Usage: python tools/energy_sweep.py '{"MOM_GROUP_M_A":"0"}' '{"MOM_GROUP_M_A":"8"}' ..."""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2504_12526_b200 import _mom  # noqa: E402

variants = [json.loads(a) for a in sys.argv[1:]] or [{}]
rounds = int(os.environ.get("ROUNDS", "3"))
iters = int(os.environ.get("ITERS", "20"))
w = synth.CONFIGS[int(os.environ.get("CFG", "1"))]
dev = torch.device("cuda:0")
d, I, S, C = w.hidden, w.intermediate, min(w.S, 65536), w.C
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, torch.bfloat16)
x = synth.hidden(S, d, dev, torch.bfloat16)
out = torch.empty_like(x)
ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S, d, I, C, torch.bfloat16), dtype=torch.uint8, device=dev)
flops = 6.0 * S * d * I
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)

acc = {i: {"tflops": [], "mhz": [], "j": []} for i in range(len(variants))}
base_env = {k: os.environ.get(k) for v in variants for k in v}
for r in range(rounds):
    for i, v in enumerate(variants):
        for k in base_env:
            os.environ.pop(k, None)
        os.environ.update(v)
        for _ in range(3):
            _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws)
        torch.cuda.synchronize()
        clocks, stop = [], threading.Event()

        def samp():
            while not stop.is_set():
                clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                time.sleep(0.01)
        t = threading.Thread(target=samp)
        t.start()
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(iters):
            _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws)
        ev1.record()
        torch.cuda.synchronize()
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        stop.set()
        t.join()
        ms = ev0.elapsed_time(ev1) / iters
        acc[i]["tflops"].append(flops / (ms * 1e-3) / 1e12)
        acc[i]["mhz"].append(statistics.mean(clocks) if clocks else float("nan"))
        acc[i]["j"].append((e1 - e0) / 1e3 / iters)
for i, v in enumerate(variants):
    a = acc[i]
    tf, mhz, j = statistics.mean(a["tflops"]), statistics.mean(a["mhz"]), statistics.mean(a["j"])
    print(json.dumps({"variant": v, "tflops": round(tf, 1), "sm_mhz": round(mhz), "joules_per_call": round(j, 3),
                      "tflop_per_joule": round(flops / 1e12 / j, 3), "tflops_per_ghz": round(tf / (mhz / 1e3), 1),
                      "rounds": [round(t, 1) for t in a["tflops"]]}), flush=True)
