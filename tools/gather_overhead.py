"""Cost of the fused all-gather stores on the compute (single GPU proxy): config-2 MLP with k
local 'peer' buffers (HBM instead of NVLink) vs the plain call; forwarding on/off."""
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
def run(k):
    if k == 0: _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws)
    else: _mom.mlp_minseq_fwd_gather(x, x, wg, wu, wd, out, peers[:k], C, ws)
res = {}
for fwd in ("1", "0"):
    os.environ["MOM_GATHER_FORWARD"] = fwd
    for k in (0, 1, 3, 7):
        if fwd == "0" and k == 0: continue
        ts = []
        for i in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(k); e1.record(); torch.cuda.synchronize()
            if i >= 2: ts.append(e0.elapsed_time(e1))
        res[f"fwd{fwd}_peers{k}"] = round(statistics.median(ts), 3)
print(json.dumps(res))
