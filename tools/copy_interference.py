"""Does PCIe DMA (KV offload D2H / reload H2D on copy engines) slow the tcgen05 MLP kernels?
Runs one config-2 mini-sequence MLP call (8 x phase A + B) while 0 / D2H / H2D / both copies of
268 MB are in flight on side streams; prints per-kernel times of the first two mini-sequences and
the mean of the rest, interleaved over rounds."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2504_12526_b200 import _mom  # noqa: E402

dev = torch.device("cuda:0")
w = synth.CONFIGS[1]
d, I, S, C = w.hidden, w.intermediate, w.S, w.C
bf = torch.bfloat16
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
x = synth.hidden(S, d, dev, bf)
out = torch.empty_like(x)
ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S, d, I, C, bf), dtype=torch.uint8, device=dev)
kv = torch.empty((S, 2 * w.d_kv), dtype=bf, device=dev).normal_()
kv_back = torch.empty_like(kv)
host_a = torch.empty(kv.shape, dtype=bf, pin_memory=True)
host_b = torch.empty(kv.shape, dtype=bf, pin_memory=True)
compute, s_d2h, s_h2d = (torch.cuda.Stream(dev) for _ in range(3))
modes = ["none", "d2h", "h2d", "both", "both_spread"]
M = (S + C - 1) // C
res = {m: [] for m in modes}
for r in range(4):
    for m in modes:
        torch.cuda.synchronize()
        timer = _mom.LaunchTimer(capacity=64)
        with timer, torch.cuda.stream(compute):
            if m in ("d2h", "both"):
                s_d2h.wait_stream(compute)
                _mom.kv_offload(kv, host_a, compute, s_d2h)
            if m in ("h2d", "both"):
                s_h2d.wait_stream(compute)
                _mom.kv_reload(host_b, kv_back, s_h2d)
            if m == "both_spread":
                # one mini-sequence per call; chunk i of each copy waits for mini-sequence i-1
                rows = kv.shape[0]
                for i in range(M):
                    if i > 0:
                        s_d2h.wait_stream(compute)
                        s_h2d.wait_stream(compute)
                    r0, r1 = i * rows // M, (i + 1) * rows // M
                    _mom.kv_offload(kv[r0:r1], host_a[r0:r1], compute, s_d2h)
                    _mom.kv_reload(host_b[r0:r1], kv_back[r0:r1], s_h2d)
                    _mom.mlp_minseq_fwd(x[i * C:(i + 1) * C], x[i * C:(i + 1) * C], wg, wu, wd,
                                        out[i * C:(i + 1) * C], C, ws, compute)
            else:
                _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws, compute)
        torch.cuda.synchronize()
        res[m].append([t for _, t in timer.results()])
for m in modes:
    runs = res[m][1:]
    a = [statistics.mean(r[k] for r in runs) for k in range(len(runs[0]))]
    print(f"{m:5s} A0 {a[0]*1e3:7.1f} B0 {a[1]*1e3:6.1f} A1 {a[2]*1e3:7.1f} B1 {a[3]*1e3:6.1f} "
          f"A2-7 {statistics.mean(a[4::2])*1e3:7.1f} B2-7 {statistics.mean(a[5::2])*1e3:6.1f} us  total {sum(a):.3f} ms")
