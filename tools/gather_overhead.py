"""Cost of the fused all-gather stores on the compute (single GPU proxy): config-2 MLP with k
local 'peer' buffers (HBM instead of NVLink) vs the plain call; forwarding on/off.  Variants are
interleaved over rounds (the power-capped clock drifts with temperature, so a fixed order biases
later variants)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom
w = synth.CONFIGS[1]; dev = torch.device("cuda:0"); bf = torch.bfloat16
d, I, S, C = w.hidden, w.intermediate, w.S, w.C
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
x = synth.hidden(S, d, dev, bf); out = torch.empty_like(x)
ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S, d, I, C, bf), dtype=torch.uint8, device=dev)
peers = [torch.empty_like(x) for _ in range(7)]
variants = [("1", 0), ("1", 1), ("1", 3), ("1", 7), ("0", 1), ("0", 3), ("0", 7)]
def run(k):
    if k == 0: _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws)
    else: _mom.mlp_minseq_fwd_gather(x, x, wg, wu, wd, out, peers[:k], C, ws)
res = {f"fwd{f}_peers{k}": [] for f, k in variants}
for r in range(int(os.environ.get("ROUNDS", "6"))):
    for fwd, k in variants:
        os.environ["MOM_GATHER_FORWARD"] = fwd
        ts = []
        for i in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(k); e1.record(); torch.cuda.synchronize()
            if i >= 2: ts.append(e0.elapsed_time(e1))
        if r > 0:
            res[f"fwd{fwd}_peers{k}"].append(statistics.median(ts))
print(json.dumps({k: round(statistics.mean(v), 3) for k, v in res.items()}))
print(json.dumps({k: [round(t, 2) for t in v] for k, v in res.items()}))
