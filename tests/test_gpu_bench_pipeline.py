"""The bench's pipelined requests (request i's KV reload overlapping request i+1's MLP, two pinned
host slots, the e2e leg's reload queued behind the next request's input rows) compute exactly what
one request computed alone: same MLP rows, same logits and token, the KV round trip intact."""
from __future__ import annotations

import os
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2504_12526_b200 import _mom  # noqa: E402

pytestmark = pytest.mark.gpu


def _reference(wl):
    """One request alone, device inputs, no overlap."""
    wg, wu, wd = wl.w0
    out = torch.empty_like(wl.x)
    _mom.mlp_minseq_fwd(wl.x, wl.x, wg, wu, wd, out, wl.C)
    wg1, wu1, wd1 = wl.w1
    y = torch.empty_like(wl.y)
    _mom.mlp_last_token(out[-1], out[-1], wg1, wu1, wd1, y)
    logits = torch.empty_like(wl.logits)
    am = torch.empty_like(wl.argmax)
    _mom.lm_head_last(y, wl.gain, wl.cfg.eps, wl.wh, logits, am)
    torch.cuda.synchronize()
    return out, logits, am


@pytest.mark.parametrize("tail", [False, True])
@pytest.mark.parametrize("e2e", [False, True])
@pytest.mark.parametrize("serial", [False, True])
def test_pipelined_steps_equal_one_request(cuda_device, e2e, serial, tail):
    cfg = synth.CONFIGS[1]
    # config-2 shapes with a shorter sequence (3 mini-sequences, ragged tail) to keep the test quick
    small = synth.Workload(cfg.name + "-test", cfg.hidden, cfg.intermediate, 2 * cfg.C + 1000, 3, 32000,
                           cfg.layers, cfg.d_kv, "bf16", cfg.eps, cfg.C)
    wl = bench.Workload(small, 0, 1, cuda_device)
    ref_out, ref_logits, ref_am = _reference(wl)
    if tail:  # request i's last-token tail on its own stream, overlapping request i+1's MLP
        wl.enable_tail_overlap()
    compute, copy, reload = (torch.cuda.Stream(cuda_device) for _ in range(3))
    h2d = torch.cuda.Stream(cuda_device)
    x_host = wl.x.cpu().pin_memory() if e2e else None
    if e2e:
        wl.init_e2e(compute)  # double-buffered device input (the second buffer starts empty)
    for o in (wl.outs if tail else [wl.out]):
        o.zero_()
    wl.kv_back.zero_()
    with torch.cuda.stream(compute):
        for _ in range(3):
            bench.run_step(wl, compute, copy, reload, [0], x_host=x_host, h2d=h2d if e2e else None, serial=serial)
        if e2e:
            bench.flush_reload(wl, h2d)
        bench.join_streams(compute, copy, reload, h2d, *wl.extra_streams())
    torch.cuda.synchronize()
    for o in (wl.outs if tail else [wl.out]):  # 3 requests: both output buffers were written
        assert torch.equal(o, ref_out)
    assert torch.equal(wl.logits, ref_logits)
    assert int(wl.argmax.item()) == int(ref_am.item())
    assert torch.equal(wl.kv_back, wl.kv)
    for slot in wl.kv_host:
        assert torch.equal(slot, wl.kv.cpu())


def test_bench_step_full_size_vs_oracle(cuda_device):
    """BASELINE config 2 at full size in exactly the bench's launch configuration (pipelined requests,
    PDL, KV copies in flight, then the e2e leg with host input): sampled output rows against the
    oracle, the last token's MLP against the oracle, and the argmax against the oracle's logits of
    the kernel's own hidden vector."""
    import oracle
    from tests.parity import TOL_BF16, assert_argmax_exact, check_close
    cfg = synth.CONFIGS[1]
    wl = bench.Workload(cfg, 0, 1, cuda_device)
    wl.enable_tail_overlap()  # bench.py --tail-overlap (the tests without it cover the default)
    compute, copy, reload = (torch.cuda.Stream(cuda_device) for _ in range(3))
    h2d = torch.cuda.Stream(cuda_device)
    x_host = wl.x.cpu().pin_memory()
    wl.init_e2e(compute)
    with torch.cuda.stream(compute):
        for _ in range(2):
            bench.run_step(wl, compute, copy, reload, [0])
        for _ in range(2):
            bench.run_step(wl, compute, copy, reload, [0], x_host=x_host, h2d=h2d)
        bench.flush_reload(wl, h2d)
        bench.join_streams(compute, copy, reload, h2d, *wl.extra_streams())
    torch.cuda.synchronize()
    rows = synth.sample_rows(wl.S, wl.C, n_random=32)
    xs = wl.x.cpu()
    wg, wu, wd = (t.cpu() for t in wl.w0)
    check_close(wl.out[rows].cpu(), oracle.mlp_rows(xs, xs, wg, wu, wd, rows), TOL_BF16, "bench step rows")
    last = wl.out[-1].cpu()
    wg1, wu1, wd1 = (t.cpu() for t in wl.w1)
    check_close(wl.y.cpu(), oracle.mlp_rows(last[None], last[None], wg1, wu1, wd1, [0])[0], TOL_BF16, "last token")
    yn = oracle.rmsnorm(wl.y.cpu().double().numpy(), wl.gain.cpu(), cfg.eps)
    ref_logits = oracle.lm_head(yn, wl.wh.cpu())[0]
    check_close(wl.logits.cpu(), ref_logits, 1e-4, "bench step LM head")
    assert_argmax_exact(int(wl.argmax.item()), ref_logits, "bench step (config 2) head")
