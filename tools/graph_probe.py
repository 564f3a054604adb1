"""CUDA-graph capture of the compute path (mini-sequence MLP, last-token MLP, LM head + argmax): replay
equals eager bitwise, and the per-step time of both (CFG = 0: config 1, fp32, launch-bound; 1: config-2 shapes)."""
import os, sys, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2504_12526_b200 import _mom
dev = torch.device("cuda:0")
CFG = int(os.environ.get("CFG", "1"))
w = synth.CONFIGS[CFG]
bf = synth.torch_dtype(w.dtype)
d, I, V, C = w.hidden, w.intermediate, w.vocab, w.C
S = w.S if CFG == 0 else 2 * C + 1000
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
wh = synth.head_weight(V, d, dev, bf); gain = synth.norm_gain(d, dev, bf)
x = synth.hidden(S, d, dev, bf)
def alloc():
    return (torch.empty_like(x), torch.empty(d, dtype=bf, device=dev), torch.empty(V, dtype=torch.float32, device=dev),
            torch.empty(1, dtype=torch.int32, device=dev))
ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S, d, I, C, bf), dtype=torch.uint8, device=dev)
def step(o):
    out, y, lg, am = o
    _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws)
    _mom.mlp_last_token(out[-1], out[-1], wg, wu, wd, y)
    _mom.lm_head_last(y, gain, 1e-5, wh, lg, am)
ref = alloc(); step(ref); torch.cuda.synchronize()
g_o = alloc()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step(g_o)  # warm-up outside capture
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
for t in g_o: t.zero_()
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g):
        step(g_o)
except Exception as e:
    print("capture failed:", type(e).__name__, str(e)[:500]); raise
for t in g_o: t.zero_()
g.replay(); torch.cuda.synchronize()
print("equal:", all(torch.equal(a, b) for a, b in zip(ref, g_o)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ("eager", "graph", "eager", "graph"):
    torch.cuda.synchronize(); e0.record()
    for _ in range(int(os.environ.get("N", "20"))):
        if mode == "graph": g.replay()
        else: step(g_o)
    e1.record(); torch.cuda.synchronize()
    print(mode, round(e0.elapsed_time(e1) / int(os.environ.get("N", "20")), 4), "ms/step")
