"""Per-launch overhead of the split (two launches per mini-sequence) schedule: the config-2 MLP
(S = 65536) with C = 8192 / 16384 / 32768 / 65536 (M = 8 / 4 / 2 / 1, 16 / 8 / 4 / 2 launches, the same
FLOPs), events around the whole call only (PDL on), variants interleaved over rounds."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom
dev = torch.device("cuda:0"); bf = torch.bfloat16
w = synth.CONFIGS[1]
d, I, S = w.hidden, w.intermediate, w.S
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
x = synth.hidden(S, d, dev, bf); out = torch.empty_like(x)
Cs = [8192, 16384, 32768, 65536]
ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S, d, I, max(Cs), bf), dtype=torch.uint8, device=dev)
res = {C: [] for C in Cs}
for r in range(int(os.environ.get("ROUNDS", "5"))):
    for C in Cs:
        ts = []
        for i in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws); e1.record(); torch.cuda.synchronize()
            if i >= 1: ts.append(e0.elapsed_time(e1))
        if r > 0: res[C].append(statistics.median(ts))
print(json.dumps({f"C={C} M={S // C}": round(statistics.mean(v), 3) for C, v in res.items()}))
print(json.dumps({f"C={C}": [round(t, 3) for t in v] for C, v in res.items()}))
