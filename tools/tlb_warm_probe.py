"""Is the last-token path slower inside a long stack because its weights' TLB entries are cold?
(config 3 shapes: W_head [152064, 3584], final-layer W_gate/W_up/W_down).  Each round first streams a
large buffer (POLLUTE_GB, default 24 GB, ~12 k distinct 2 MB pages, like a stack's other layers), then
times mom_mlp_last_token + mom_lm_head_last with CUDA events, either directly ("cold") or after a
page-touch pass over their weights (one 4-byte load per 64 KB, a strided torch gather: "touched").
Also a "warm" reference: the same calls repeated back to back."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom

w = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
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
gb = float(os.environ.get("POLLUTE_GB", "24"))
pol_a = torch.empty(int(gb * 1e9 / 2) // 4, dtype=torch.int32, device=dev)
pol_b = torch.empty_like(pol_a)


def touch(ts):
    for t in ts:
        t.view(-1).view(torch.int32)[:: 16384].sum()  # one 4-B load per 64 KB


def timed():
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    _mom.mlp_last_token(x, x, wg, wu, wd, y)
    e[1].record()
    _mom.lm_head_last(y, gain, w.eps, wh, logits, am)
    e[2].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) * 1e3, e[1].elapsed_time(e[2]) * 1e3


res = {"workload": w.name, "pollute_gb": gb}
for mode in ("cold", "touched", "cold", "touched", "warm"):
    lt, hd = [], []
    for i in range(8):
        if mode != "warm":
            pol_b.copy_(pol_a)
            if mode == "touched":
                touch([wg, wu, wd, wh])
        torch.cuda.synchronize()
        a, b = timed()
        lt.append(a)
        hd.append(b)
    key = mode if mode not in res else mode + "_2"
    res[key] = {"last_token_us": round(statistics.median(lt), 1), "lm_head_us": round(statistics.median(hd), 1),
                "lm_head_tbs": round(V * d * 2 / (statistics.median(hd) * 1e-6) / 1e12, 2),
                "last_token_tbs": round(3 * d * I * 2 / (statistics.median(lt) * 1e-6) / 1e12, 2)}
print(json.dumps(res))
