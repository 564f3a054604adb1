"""LM head (config 4 shapes) timed alone and with a concurrent pinned-host copy on another stream
(D2H 2 GB, or H2D 2 GB) -- do the copy engines' HBM accesses slow the HBM-bound head?"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom

w = synth.CONFIGS[int(os.environ.get("CFG", "3"))]
dev = torch.device("cuda:0")
bf = torch.bfloat16
d, V = w.hidden, w.vocab
wh = synth.head_weight(V, d, dev, bf)
gain = synth.norm_gain(d, dev, bf)
y = synth.hidden(1, d, dev, bf)[0]
logits = torch.empty(V, dtype=torch.float32, device=dev)
am = torch.empty(1, dtype=torch.int32, device=dev)
n = 1 << 30
dbuf = torch.empty(n, dtype=bf, device=dev)
hbuf = torch.empty(n, dtype=bf, pin_memory=True)
cp = torch.cuda.Stream()
res = {"workload": w.name}
for mode in ("alone", "d2h", "h2d", "alone", "d2h", "h2d"):
    ts = []
    for i in range(10):
        torch.cuda.synchronize()
        if mode == "d2h":
            with torch.cuda.stream(cp):
                hbuf.copy_(dbuf, non_blocking=True)
        elif mode == "h2d":
            with torch.cuda.stream(cp):
                dbuf.copy_(hbuf, non_blocking=True)
        torch.cuda._sleep(2_000_000)  # ~1 ms: the copy is streaming when the head starts
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _mom.lm_head_last(y, gain, w.eps, wh, logits, am)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    t = statistics.median(ts)
    res.setdefault(mode, []).append({"us": round(t, 1), "tbs": round(V * d * 2 / (t * 1e-6) / 1e12, 2)})
print(json.dumps(res))
