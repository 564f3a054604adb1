"""One config-2 mini-sequence (S = C = 8192 rows, d 4096, I 14336) through mom_mlp_minseq_fwd, twice
(the first call warms up); for ncu captures of a single phase-A / phase-B launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom

w = synth.CONFIGS[1]
dev = torch.device("cuda:0")
bf = torch.bfloat16
wg, wu, wd = synth.mlp_weights(w.hidden, w.intermediate, 0, dev, bf)
x = synth.hidden(w.C, w.hidden, dev, bf)
out = torch.empty_like(x)
for _ in range(2):
    _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, w.C)
torch.cuda.synchronize()
print("ok")
