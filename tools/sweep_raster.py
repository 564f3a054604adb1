"""Sweep the tcgen05 kernels' raster group (MOM_GROUP_M_A / MOM_GROUP_M_B) and CTA group at
config 2 shapes; prints per-phase ms and TFLOP/s (CUDA events on the launching stream)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom

w = synth.CONFIGS[1]
dev = torch.device("cuda:0")
d, I, S, C = w.hidden, w.intermediate, w.S, w.C
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, torch.bfloat16)
x = synth.hidden(S, d, dev, torch.bfloat16)
out = torch.empty_like(x)
ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S, d, I, C, torch.bfloat16), dtype=torch.uint8, device=dev)
M = S // C
timer = _mom.LaunchTimer(capacity=4 * M * 8)
configs = [dict(MOM_GROUP_M_A=a, MOM_GROUP_M_B=b, MOM_CTA_GROUP=cg)
           for cg in sys.argv[1:2] or ["2"]
           for a in ["0", "16", "8", "4"] for b in ["8"]] + \
          [dict(MOM_GROUP_M_A="0", MOM_GROUP_M_B=b, MOM_CTA_GROUP="2") for b in ["1", "2", "4", "16", "32"]]
res = []
for cfg in configs:
    os.environ.update(cfg)
    for _ in range(2):
        _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws)
    torch.cuda.synchronize()
    with timer:
        for _ in range(3):
            _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws)
        torch.cuda.synchronize()
    per = {}
    for k, t in timer.results():
        per.setdefault(k, []).append(t)
    ta, tb = statistics.mean(per["phaseA_tc"]), statistics.mean(per["phaseB_tc"])
    r = dict(cfg, a_ms=round(ta, 4), b_ms=round(tb, 4), a_tflops=round(4 * C * d * I / ta / 1e9, 1),
             b_tflops=round(2 * C * d * I / tb / 1e9, 1), mlp_tflops=round(6 * S * d * I / (M * (ta + tb)) / 1e9, 1))
    print(json.dumps(r), flush=True)
