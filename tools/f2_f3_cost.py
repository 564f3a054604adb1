"""One-GPU measurements of two NEXT rows:
f2 -- the vocab-sharded LM head: time of one rank's shard (V/N rows of W_head + packed-key argmax) at
      N = 1, 2, 4, 8 (the cross-rank u64 max is one 8-byte NCCL all-reduce, not measurable here);
f3 -- the per-layer RMSNorm folded into phase A: config-2 mini-sequence MLP (x + MLP(norm(x))) with the
      gain folded into W_gate/W_up and 1/rms applied in the phase-A epilogue, vs the plain MLP call
      (x + MLP(x)), and vs an unfused torch RMSNorm pass followed by the plain call.
CUDA events (a GPU sleep queued first, so the host's per-call overhead is not in the interval), median of
10 after 3 warm-ups, config 2 shapes."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom

w = synth.CONFIGS[1]
dev = torch.device("cuda:0")
bf = torch.bfloat16
d, I, V, C = w.hidden, w.intermediate, w.vocab, w.C


def timeit(fn, n=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(1_000_000)  # the GPU waits while the host enqueues: host call overhead not timed
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


res = {"workload": w.name}
wh = synth.head_weight(V, d, dev, bf)
gain = synth.norm_gain(d, dev, bf)
y = synth.hidden(1, d, dev, bf)[0]
key = torch.zeros(1, dtype=torch.int64, device=dev)
for N in (1, 2, 4, 8):
    per = -(-V // N)
    lg = torch.empty(per, dtype=torch.float32, device=dev)
    ms = timeit(lambda: _mom.lm_head_shard(y, gain, w.eps, wh[:per], 0, lg, key))
    res[f"f2_head_shard_N{N}_us"] = round(ms * 1e3, 1)
    res[f"f2_head_shard_N{N}_tbs"] = round(per * d * 2 / (ms * 1e-3) / 1e12, 2)
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
x = (synth.hidden(C, d, dev, torch.float32) * 3.0).to(bf)
out = torch.empty_like(x)
ws = torch.empty(_mom.lib().mom_mlp_minseq_rmsnorm_workspace_bytes(C, d, I, C, 0), dtype=torch.uint8, device=dev)
wgf, wuf = _mom.fold_norm_gain(wg, gain), _mom.fold_norm_gain(wu, gain)
plain = timeit(lambda: _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws))
folded = timeit(lambda: _mom.mlp_minseq_rmsnorm_fwd(x, wgf, wuf, wd, out, C, w.eps, ws))
xn = torch.empty_like(x)


def unfused():
    xf = x.float()
    xn.copy_((xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + w.eps) * gain.float()).to(bf))
    _mom.mlp_minseq_fwd(xn, x, wg, wu, wd, out, C, ws)


unf = timeit(unfused)
fold_once = timeit(lambda: (_mom.fold_norm_gain(wg, gain, wgf), _mom.fold_norm_gain(wu, gain, wuf)), n=5)
res.update({"f3_plain_mlp_ms": round(plain, 3), "f3_folded_norm_mlp_ms": round(folded, 3),
            "f3_torch_norm_then_mlp_ms": round(unf, 3), "f3_overhead_pct": round(100 * (folded / plain - 1), 2),
            "f3_fold_gain_once_per_layer_ms": round(fold_once, 3)})
print(json.dumps(res))
