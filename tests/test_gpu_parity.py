"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs (synth/), plus the exact GPU-only invariants.  All tests need a B200: -m gpu.

Bars (BASELINE.json north_star):
  bf16 MLP: normwise max relative error <= 2e-2 per tensor and per row;
  (and <= 6e-3 regression bound, tests/parity.py);  fp32 MLP: <= 1e-4;  argmax: bit-exact
  (against the oracle's argmax of the kernel's fp32 logits AND of the float64 oracle's logits,
  top-2 gap logged);  bit-identity across mini-sequence counts; KV round trip exact.
"""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2504_12526_b200 import _mom
from tests.parity import TOL_BF16, TOL_F32, assert_argmax_exact, check_close

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cta_group_env():
    old = os.environ.get("MOM_CTA_GROUP")
    yield
    if old is None:
        os.environ.pop("MOM_CTA_GROUP", None)
    else:
        os.environ["MOM_CTA_GROUP"] = old


def _mlp_inputs(S, d, I, dtype, device, layer=0, residual=True):
    wg, wu, wd = synth.mlp_weights(d, I, layer, "cpu", dtype)
    x = synth.hidden(S, d, "cpu", dtype)
    res = synth.hidden(S, d, "cpu", dtype, seed=synth.SEED_X + 1) if residual else None
    dev = lambda t: None if t is None else t.to(device)  # noqa: E731
    return (x, res, wg, wu, wd), tuple(dev(t) for t in (x, res, wg, wu, wd))


def _run_fwd(gx, gres, gwg, gwu, gwd, C, out=None):
    out = torch.empty_like(gx) if out is None else out
    _mom.mlp_minseq_fwd(gx, gres, gwg, gwu, gwd, out, C)
    torch.cuda.synchronize()
    return out


# ------------------------------------------------------------------ config 1 (fp32 SIMT)
def test_cfg1_f32_full_tensor(cuda_device):
    w = synth.CONFIGS[0]
    (x, res, wg, wu, wd), g = _mlp_inputs(w.S, w.hidden, w.intermediate, torch.float32, cuda_device)
    out = _run_fwd(*g, C=w.C)
    ref = oracle.mlp_minseq(x, res, wg, wu, wd, C=w.C)
    check_close(out, ref, TOL_F32, "cfg1 f32 with residual")
    out0 = _run_fwd(g[0], None, *g[2:], C=w.C)  # Alg. 1's O_i = MLP(A_i), no residual
    ref0 = oracle.mlp_minseq(x, None, wg, wu, wd, C=w.C)
    check_close(out0, ref0, TOL_F32, "cfg1 f32 no residual")
    for C in (1, 7, 1000, w.S, w.S + 5):  # bit-identity across M on the GPU
        assert torch.equal(_run_fwd(*g, C=C), out), C


# ------------------------------------------------------------------ bf16 tcgen05, small + ragged
@pytest.mark.parametrize("cta_group", ["1", "2"])
@pytest.mark.parametrize("S,d,I,C", [(1024, 256, 688, 256), (1000, 512, 1024, 300), (77, 256, 384, 64),
                                     (300, 384, 640, 300)])
def test_bf16_tcgen05_vs_oracle(cuda_device, cta_group, S, d, I, C):
    os.environ["MOM_CTA_GROUP"] = cta_group
    (x, res, wg, wu, wd), g = _mlp_inputs(S, d, I, torch.bfloat16, cuda_device)
    out = _run_fwd(*g, C=C)
    ref = oracle.mlp_minseq(x, res, wg, wu, wd, C=C)
    check_close(out, ref, TOL_BF16, f"bf16 S={S} d={d} I={I} C={C} cg={cta_group}")
    out0 = _run_fwd(g[0], None, *g[2:], C=C)
    ref0 = oracle.mlp_minseq(x, None, wg, wu, wd, C=C)
    check_close(out0, ref0, TOL_BF16, "bf16 no residual")


@pytest.mark.parametrize("cta_group", ["1", "2"])
def test_bf16_bit_identical_across_M(cuda_device, cta_group):
    """P:286 identical logits <- P:109-113 row partition: GPU output bitwise equal for every C."""
    os.environ["MOM_CTA_GROUP"] = cta_group
    S, d, I = 1000, 256, 688
    _, g = _mlp_inputs(S, d, I, torch.bfloat16, cuda_device)
    ref = _run_fwd(*g, C=S)
    for C in (1, 100, 128, 129, 256, 333, 999, S + 7):
        assert torch.equal(_run_fwd(*g, C=C), ref), C


def test_bf16_cta_groups_agree(cuda_device):
    S, d, I = 700, 512, 1536
    _, g = _mlp_inputs(S, d, I, torch.bfloat16, cuda_device)
    os.environ["MOM_CTA_GROUP"] = "1"
    a = _run_fwd(*g, C=256)
    os.environ["MOM_CTA_GROUP"] = "2"
    b = _run_fwd(*g, C=256)
    assert torch.equal(a, b)


def test_bf16_in_place(cuda_device):
    """out may alias residual and x (the layer loop's x_{l+1} = x_l + MLP(x_l))."""
    S, d, I = 640, 256, 512
    (x, _, wg, wu, wd), g = _mlp_inputs(S, d, I, torch.bfloat16, cuda_device, residual=False)
    gx = g[0].clone()
    ref = _run_fwd(g[0], g[0], *g[2:], C=200)
    _mom.mlp_minseq_fwd(gx, gx, g[2], g[3], g[4], gx, 200)
    torch.cuda.synchronize()
    assert torch.equal(gx, ref)


# ------------------------------------------------------------------ config 2 at full size
def test_cfg2_llama_full_size_sampled_rows(cuda_device):
    """BASELINE config 2 (d=4096, I=14336, S=65536, M=8) in the bench's launch configuration;
    the oracle checks sampled rows (random + 0, S-1 and both sides of every boundary)."""
    w = synth.CONFIGS[1]
    wg, wu, wd = synth.mlp_weights(w.hidden, w.intermediate, 0, cuda_device, torch.bfloat16)
    x = synth.hidden(w.S, w.hidden, cuda_device, torch.bfloat16)
    out = torch.empty_like(x)
    _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, w.C)
    torch.cuda.synchronize()
    rows = synth.sample_rows(w.S, w.C, n_random=96)
    xs = x.cpu()
    ref = oracle.mlp_rows(xs, xs, wg.cpu(), wu.cpu(), wd.cpu(), rows)
    check_close(out[rows].cpu(), ref, TOL_BF16, "cfg2 sampled rows")


# ------------------------------------------------------------------ last token + LM head
@pytest.mark.parametrize("cfg", [0, 1])
def test_last_token_mlp_and_lm_head(cuda_device, cfg):
    w = synth.CONFIGS[cfg]
    dt = synth.torch_dtype(w.dtype)
    d, I, V = w.hidden, w.intermediate, w.vocab
    wg, wu, wd = synth.mlp_weights(d, I, 0, "cpu", dt)
    wh = synth.head_weight(V, d, "cpu", dt)
    gain = synth.norm_gain(d, "cpu", dt)
    x = synth.hidden(4, d, "cpu", dt)  # rows of the final layer's input; the last one is used
    res = synth.hidden(4, d, "cpu", dt, seed=synth.SEED_X + 1)
    G = lambda t: t.to(cuda_device)  # noqa: E731
    y = torch.empty(d, dtype=dt, device=cuda_device)
    _mom.mlp_last_token(G(x)[3], G(res)[3], G(wg), G(wu), G(wd), y)
    logits = torch.empty(V, dtype=torch.float32, device=cuda_device)
    am = torch.empty(1, dtype=torch.int32, device=cuda_device)
    _mom.lm_head_last(y, G(gain), w.eps, G(wh), logits, am)
    torch.cuda.synchronize()
    tol = TOL_F32 if w.dtype == "f32" else TOL_BF16
    y_ref = oracle.mlp_rows(x, res, wg, wu, wd, [3])[0]
    check_close(y.cpu(), y_ref, tol, "last-token MLP")
    # LM head checked on the GPU's own hidden vector (same input to both sides)
    yn = oracle.rmsnorm(y.cpu().double().numpy(), gain, w.eps)
    ref_logits = oracle.lm_head(yn, wh)[0]
    check_close(logits.cpu(), ref_logits, 1e-4, "lm head logits")
    # argmax: bit-exact on the kernel's fp32 logits and against the float64 oracle's logits
    assert int(am.item()) == oracle.argmax_f32(logits.cpu().numpy())
    assert_argmax_exact(int(am.item()), ref_logits, f"cfg{cfg + 1} last-token head")
    # no-norm variant and logits=NULL variant give the same argmax as their logits
    _mom.lm_head_last(y, None, 0.0, G(wh), logits, am)
    am2 = torch.empty(1, dtype=torch.int32, device=cuda_device)
    _mom.lm_head_last(y, None, 0.0, G(wh), None, am2)
    torch.cuda.synchronize()
    assert int(am.item()) == int(am2.item()) == oracle.argmax_f32(logits.cpu().numpy())
    check_close(logits.cpu(), oracle.lm_head(y.cpu().double().numpy(), wh)[0], 1e-4, "lm head no norm")


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_lm_head_eps_placement(cuda_device, dt):
    """S:126 eps inside the square root, pinned through the kernel: with eps = 3 on a unit-RMS hidden
    vector 1/sqrt(1 + 3) = 0.5 exactly, while eps outside the root gives 0.25 and eps dropped 1.0, so a
    misplaced eps scales every logit by 2 or 1/2.  A +-1 vector has mean(h^2) = 1 exactly."""
    d, V = 512, 3000
    g = torch.Generator().manual_seed(5)
    h = torch.where(torch.rand(d, generator=g) < 0.5, -1.0, 1.0).to(dt)
    wh = synth.head_weight(V, d, "cpu", dt)
    gain = synth.norm_gain(d, "cpu", dt)
    G = lambda t: t.to(cuda_device)  # noqa: E731
    logits = torch.empty(V, dtype=torch.float32, device=cuda_device)
    am = torch.empty(1, dtype=torch.int32, device=cuda_device)
    for eps in (3.0, 0.0):
        _mom.lm_head_last(G(h), G(gain), eps, G(wh), logits, am)
        torch.cuda.synchronize()
        hn = h.double().numpy() * (1.0 / np.sqrt(1.0 + eps)) * gain.double().numpy()  # closed form
        assert np.array_equal(oracle.rmsnorm(h.double().numpy(), gain, eps), hn)
        ref = oracle.lm_head(hn, wh)[0]
        check_close(logits.cpu(), ref, 1e-4, f"lm head eps={eps}")
        assert_argmax_exact(int(am.item()), ref, f"lm head eps={eps}")


def test_rmsnorm_folded_eps_placement(cuda_device):
    """The f3 path's row 1/rms (norm.cu) with eps = 3 on +-1 rows (mean(x^2) = 1): the MLP input is
    x / 2 * gain; against the oracle's literal norm-then-MLP.  eps outside the root would feed x / 4."""
    S, d, I, C = 300, 256, 512, 128
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, "cpu", bf)
    gain = torch.ones(d, dtype=bf)
    g = torch.Generator().manual_seed(6)
    x = torch.where(torch.rand(S, d, generator=g) < 0.5, -1.0, 1.0).to(bf)
    G = lambda t: t.to(cuda_device)  # noqa: E731
    out = torch.empty((S, d), dtype=bf, device=cuda_device)
    _mom.mlp_minseq_rmsnorm_fwd(G(x), G(wg), G(wu), G(wd), out, C, 3.0)
    torch.cuda.synchronize()
    rows = list(range(S))
    ref = oracle.mlp_norm_rows(x, gain, 3.0, wg, wu, wd, rows)
    check_close(out.cpu(), ref, TOL_BF16, "folded RMSNorm eps=3")
    half = (x.float() * 0.5).to(bf)  # exact: the normed rows are x / 2
    check_close(out.cpu(), oracle.mlp_rows(half, x, wg, wu, wd, rows), TOL_BF16, "folded RMSNorm eps=3 vs x/2")


def test_argmax_ties_lowest_index(cuda_device):
    """S:333 tie at 2 and 5 -> 2, through the real kernel: identity head, h with equal maxima."""
    d, V = 64, 96
    wh = torch.zeros(V, d, dtype=torch.bfloat16)
    for i in range(d):
        wh[i, i] = 1.0
    h = torch.zeros(d, dtype=torch.bfloat16)
    h[2] = h[5] = h[40] = 3.0
    logits = torch.empty(V, dtype=torch.float32, device=cuda_device)
    am = torch.empty(1, dtype=torch.int32, device=cuda_device)
    _mom.lm_head_last(h.to(cuda_device), None, 0.0, wh.to(cuda_device), logits, am)
    torch.cuda.synchronize()
    assert int(am.item()) == 2
    h[:] = -2.0
    h[63] = -1.5  # logits -2 / -1.5 on the identity rows 0..63, exactly 0 on the zero rows 64..95
    _mom.lm_head_last(h.to(cuda_device), None, 0.0, wh.to(cuda_device), logits, am)
    torch.cuda.synchronize()
    assert int(am.item()) == 64  # a 32-way tie at 0.0 -> the lowest index
    wh[95, 0] = -1.0  # row 95: logit +2.0, the unique max
    _mom.lm_head_last(h.to(cuda_device), None, 0.0, wh.to(cuda_device), logits, am)
    torch.cuda.synchronize()
    assert int(am.item()) == 95


def test_last_token_matches_full_sequence_last_row(cuda_device):
    """Alg. 1 final branch vs the standard path: GEMV last-token MLP == last row of the
    mini-sequence MLP within the bf16 bar (both compared to the same oracle row)."""
    S, d, I = 300, 512, 1024
    (x, res, wg, wu, wd), g = _mlp_inputs(S, d, I, torch.bfloat16, cuda_device)
    full = _run_fwd(*g, C=128)
    y = torch.empty(d, dtype=torch.bfloat16, device=cuda_device)
    _mom.mlp_last_token(g[0][S - 1], g[1][S - 1], g[2], g[3], g[4], y)
    torch.cuda.synchronize()
    ref = oracle.mlp_rows(x, res, wg, wu, wd, [S - 1])[0]
    check_close(y.cpu(), ref, TOL_BF16, "last token")
    check_close(full[S - 1].cpu(), ref, TOL_BF16, "full last row")


# ------------------------------------------------------------------ KV offload / reload
def test_kv_offload_reload_roundtrip(cuda_device):
    """Alg. 1 P:99 / P:106: bytewise round trip; ledger D2H = H2D = 2*S*d_kv*L*w (Eq. 2)."""
    S, d_kv, L = 4096, 1024, 3
    kv = [synth.kv_standin(S, d_kv, l, cuda_device) for l in range(L)]
    host = [torch.empty_like(k, device="cpu").pin_memory() for k in kv]
    back = [torch.empty_like(k) for k in kv]
    prod = torch.cuda.current_stream()
    cp = torch.cuda.Stream()
    d2h = h2d = 0
    for l in range(L):
        done = torch.cuda.Event()
        _mom.kv_offload(kv[l], host[l], prod, cp, done)
        d2h += kv[l].numel() * kv[l].element_size()
    cp.synchronize()
    for l in range(L):
        _mom.kv_reload(host[l], back[l], cp)
        h2d += kv[l].numel() * kv[l].element_size()
    cp.synchronize()
    for l in range(L):
        assert torch.equal(host[l], kv[l].cpu())
        assert torch.equal(back[l], kv[l])
    assert d2h == h2d == 2 * S * d_kv * L * 2


def test_kv_offload_rejects_pageable_host(cuda_device):
    kv = torch.zeros(1024, dtype=torch.bfloat16, device=cuda_device)
    host = torch.empty(1024, dtype=torch.bfloat16)  # not pinned
    with pytest.raises(_mom.MomError) as ei:
        _mom.kv_offload(kv, host)
    assert ei.value.status == _mom.MOM_ERR_INVALID_ARG


def test_workspace_too_small_is_reported(cuda_device):
    S, d, I = 256, 256, 512
    _, g = _mlp_inputs(S, d, I, torch.bfloat16, cuda_device)
    ws = torch.empty(1024, dtype=torch.uint8, device=cuda_device)
    with pytest.raises(_mom.MomError) as ei:
        _mom.mlp_minseq_fwd(*g, torch.empty_like(g[0]), 128, workspace=ws)
    assert ei.value.status == _mom.MOM_ERR_WORKSPACE


def test_from_host_streamed_equals_device_input(cuda_device):
    """mom_mlp_minseq_fwd_from_host (per-mini-sequence H2D overlapped with the MLP) gives the
    bitwise result of the device-input call, for ragged mini-sequences."""
    S, d, I, C = 1000, 256, 688, 300
    (x, res, wg, wu, wd), g = _mlp_inputs(S, d, I, torch.bfloat16, cuda_device, residual=False)
    ref = _run_fwd(g[0], g[0], *g[2:], C=C)
    x_host = x.pin_memory()
    x_dev = torch.zeros_like(g[0])
    out = torch.empty_like(g[0])
    cp = torch.cuda.Stream()
    _mom.mlp_minseq_fwd_from_host(x_host, x_dev, x_dev, g[2], g[3], g[4], out, C, copy_stream=cp)
    torch.cuda.synchronize()
    assert torch.equal(x_dev, g[0])
    assert torch.equal(out, ref)
    with pytest.raises(_mom.MomError):  # pageable host memory is rejected
        _mom.mlp_minseq_fwd_from_host(x.clone(), x_dev, x_dev, g[2], g[3], g[4], out, C, copy_stream=cp)


def test_from_host_prefetch_double_buffered(cuda_device):
    """x_free (prefetch): consecutive requests alternate two device input buffers and each
    request's H2D waits only for the request that last used its buffer, so it streams in while the
    previous request computes.  Every request's output equals the device-input call bitwise."""
    S, d, I, C = 1000, 256, 688, 300
    (x, res, wg, wu, wd), g = _mlp_inputs(S, d, I, torch.bfloat16, cuda_device, residual=False)
    xs = [x, (x * -0.5).to(torch.bfloat16), (x * 2).to(torch.bfloat16)]
    refs = []
    for xi in xs:
        xd = xi.to(cuda_device)
        refs.append(_run_fwd(xd, xd, *g[2:], C=C))
    hosts = [xi.pin_memory() for xi in xs]
    bufs = [torch.zeros_like(g[0]) for _ in range(2)]
    outs = [torch.empty_like(g[0]) for _ in range(6)]
    free = [torch.cuda.Event() for _ in range(2)]
    compute, cp = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(compute):
        for e in free:
            e.record(compute)
        for r in range(6):
            slot = r % 2
            _mom.mlp_minseq_fwd_from_host(hosts[r % 3], bufs[slot], bufs[slot], g[2], g[3], g[4], outs[r], C,
                                          stream=compute, copy_stream=cp, x_free=free[slot])
            free[slot].record(compute)
    torch.cuda.synchronize()
    for r in range(6):
        assert torch.equal(outs[r], refs[r % 3]), r


# ------------------------------------------------------------------ f3: RMSNorm folded into phase A
@pytest.mark.parametrize("S,d,I,C", [(1000, 512, 1024, 300), (4096, 4096, 14336, 2048)])
def test_rmsnorm_folded_mlp(cuda_device, S, d, I, C):
    """out = x + MLP(RMSNorm(x) * g) with g folded into W_gate/W_up and 1/rms applied to the
    phase-A accumulators, against the oracle's literal norm-then-MLP."""
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, "cpu", bf)
    gain = synth.norm_gain(d, "cpu", bf)
    x = (synth.hidden(S, d, "cpu", torch.float32) * 3.0).to(bf)  # un-normed residual stream, rms ~ 3
    eps = 1e-5
    G = lambda t: t.to(cuda_device)  # noqa: E731
    wg_f = _mom.fold_norm_gain(G(wg), G(gain))
    wu_f = _mom.fold_norm_gain(G(wu), G(gain))
    torch.cuda.synchronize()
    assert torch.equal(wg_f.cpu(), (wg.float() * gain.float()).to(bf))  # RNE of w * g
    out = torch.empty((S, d), dtype=bf, device=cuda_device)
    _mom.mlp_minseq_rmsnorm_fwd(G(x), wg_f, wu_f, G(wd), out, C, eps)
    torch.cuda.synchronize()
    rows = synth.sample_rows(S, C, n_random=64) if S > 1000 else list(range(S))
    ref = oracle.mlp_norm_rows(x, gain, eps, wg, wu, wd, rows)
    check_close(out[rows].cpu(), ref, TOL_BF16, "folded RMSNorm MLP")
    gx = G(x)
    _mom.mlp_minseq_rmsnorm_fwd(gx, wg_f, wu_f, G(wd), gx, C, eps)  # in place
    torch.cuda.synchronize()
    assert torch.equal(gx, out)


@pytest.mark.parametrize("d,I", [(4096, 14336), (520, 1160)])
def test_last_token_rmsnorm_vs_oracle(cuda_device, d, I):
    """f3 on the last token (mom_mlp_last_token_rmsnorm): out = x + MLP(RMSNorm(x) * g) with g folded into
    W_gate / W_up and the norm applied to the GEMV's staged x; against the oracle's literal norm-then-MLP
    (S:126), and equal to the tcgen05 folded-norm path's row within the bf16 bar."""
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, "cpu", bf)
    gain = synth.norm_gain(d, "cpu", bf)
    x = (synth.hidden(3, d, "cpu", torch.float32) * 3.0).to(bf)
    G = lambda t: t.to(cuda_device)  # noqa: E731
    wg_f, wu_f = _mom.fold_norm_gain(G(wg), G(gain)), _mom.fold_norm_gain(G(wu), G(gain))
    for eps in (1e-5, 3.0):
        y = torch.empty(d, dtype=bf, device=cuda_device)
        _mom.mlp_last_token_rmsnorm(G(x)[2], wg_f, wu_f, G(wd), y, eps)
        torch.cuda.synchronize()
        ref = oracle.mlp_norm_rows(x, gain, eps, wg, wu, wd, [2])[0]
        check_close(y.cpu(), ref, TOL_BF16, f"last-token rmsnorm d={d} I={I} eps={eps}")
    with pytest.raises(_mom.MomError):
        _mom.mlp_last_token_rmsnorm(G(x)[2], wg_f, wu_f, G(wd), y, -1.0)
