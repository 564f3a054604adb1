"""Small tcgen05 MLP calls for compute-sanitizer: ragged mini-sequences with phase-A half-width tail
tiles (S=2000, C=600, I=4096), both CTA-group modes, the fused single-launch mode, the f1 gather into
two local peer buffers, plus the last-token GEMVs, the LM head and the fp32 SIMT path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom

dev = torch.device("cuda:0")
bf = torch.bfloat16
S, d, I, C = 2000, 512, 4096, 600
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
x = synth.hidden(S, d, dev, bf)
for cg in ("2", "1"):
    os.environ["MOM_CTA_GROUP"] = cg
    out = torch.empty_like(x)
    _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C)
    torch.cuda.synchronize()
# fused single-launch mode (phase-B producers acquire phase-A row-block counters)
os.environ["MOM_CTA_GROUP"] = "2"
os.environ["MOM_FUSED"] = "1"
out_f = torch.empty_like(x)
_mom.mlp_minseq_fwd(x, x, wg, wu, wd, out_f, C)
torch.cuda.synchronize()
os.environ["MOM_FUSED"] = "0"
# f1 gather: rank 1 of 3 with two local "peer" buffers (forwarding warps + epilogue peer stores)
peers = [torch.zeros(3 * S, d, dtype=bf, device=dev) for _ in range(2)]
mine = torch.zeros(3 * S, d, dtype=bf, device=dev)
_mom.mlp_minseq_fwd_gather(x, x, wg, wu, wd, mine[S:2 * S], [p[S:2 * S] for p in peers], C)
torch.cuda.synchronize()
assert torch.equal(out_f, out) and all(torch.equal(p[S:2 * S], out) for p in peers + [mine])
y = torch.empty(d, dtype=bf, device=dev)
_mom.mlp_last_token(out[-1], out[-1], wg, wu, wd, y)
# f3: folded RMSNorm in the MLP and in the last-token GEMV
g = synth.norm_gain(d, dev, bf)
wgf, wuf = _mom.fold_norm_gain(wg, g), _mom.fold_norm_gain(wu, g)
out_n = torch.empty_like(x)
_mom.mlp_minseq_rmsnorm_fwd(x, wgf, wuf, wd, out_n, C, 1e-5)
y_n = torch.empty(d, dtype=bf, device=dev)
_mom.mlp_last_token_rmsnorm(x[-1], wgf, wuf, wd, y_n, 1e-5)
torch.cuda.synchronize()
wh = synth.head_weight(1000, d, dev, bf)
logits = torch.empty(1000, dtype=torch.float32, device=dev)
am = torch.empty(1, dtype=torch.int32, device=dev)
_mom.lm_head_last(y, synth.norm_gain(d, dev, bf), 1e-5, wh, logits, am)
torch.cuda.synchronize()
# fp32 SIMT path (double-buffered K tiles, ragged K tail: I = 688 is not a multiple of the 32-wide K tile)
d32, I32 = 256, 688
wg32, wu32, wd32 = synth.mlp_weights(d32, I32, 0, dev, torch.float32)
x32 = synth.hidden(300, d32, dev, torch.float32)
out32 = torch.empty_like(x32)
_mom.mlp_minseq_fwd(x32, x32, wg32, wu32, wd32, out32, 128)
torch.cuda.synchronize()
print("sanitize case OK", float(out.float().abs().mean()), int(am.item()), float(out32.abs().mean()))
