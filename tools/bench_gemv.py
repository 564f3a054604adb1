"""GEMV kernels of the last-token path in isolation (config 2 shapes): last-token MLP pair
(3*d*I*2 bytes of weights) and LM head (V*d*2 bytes), CUDA events, L2 flushed between calls
(HOT=1: each call right after a one-mini-sequence MLP call instead, as inside the bench step)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom

w = synth.CONFIGS[int(os.environ.get("CFG", "1"))]
dev = torch.device("cuda:0")
bf = torch.bfloat16
d, I, V = w.hidden, w.intermediate, w.vocab
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
wh = synth.head_weight(V, d, dev, bf)
gain = synth.norm_gain(d, dev, bf)
x = synth.hidden(1, d, dev, bf)[0]
y = torch.empty(d, dtype=bf, device=dev)
logits = torch.empty(V, dtype=torch.float32, device=dev)
am = torch.empty(1, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
except OSError:
    peak = 6650.0  # B200_PROFILING.md fallback
hot = os.environ.get("HOT", "0") == "1"
if hot:
    xs = synth.hidden(w.C, d, dev, bf)
    outs = torch.empty_like(xs)
    ws = torch.empty(_mom.mlp_minseq_workspace_bytes(w.C, d, I, w.C, bf), dtype=torch.uint8, device=dev)
res = {"mode": "hot (after an MLP call)" if hot else "cold (L2 flushed)"}
for name, fn, nbytes in (("last_token_mlp", lambda: _mom.mlp_last_token(x, x, wg, wu, wd, y), 3 * d * I * 2),
                         ("lm_head", lambda: _mom.lm_head_last(y, gain, w.eps, wh, logits, am), V * d * 2)):
    ts = []
    for i in range(25):
        if hot:  # as in the bench step: right after a tcgen05 MLP call (loaded clock, L2 full of MLP data)
            _mom.mlp_minseq_fwd(xs, xs, wg, wu, wd, outs, w.C, ws)
        else:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1))
    t = statistics.median(ts)
    res[name] = {"us": round(t * 1e3, 1), "gbs": round(nbytes / (t * 1e-3) / 1e9, 1), "frac_hbm": round(nbytes / (t * 1e-3) / 1e9 / peak, 3)}
print(json.dumps(res))
