"""Randomised shapes through the tcgen05 path (seeded, so reproducible): hidden and intermediate any
multiple of 8 (the 16-byte TMA pitch rule), S and C arbitrary.  Every draw is checked against the
oracle on all rows, and against itself for bit-identity across a second, different C."""
from __future__ import annotations

import random

import pytest
import torch

import oracle
import synth
from paper_2504_12526_b200 import _mom
from tests.parity import TOL_BF16, check_close

pytestmark = pytest.mark.gpu


def _draws(n, seed=123):
    rnd = random.Random(seed)
    for _ in range(n):
        d = 8 * rnd.randint(2, 96)      # 16 .. 768
        I = 8 * rnd.randint(2, 160)     # 16 .. 1280
        S = rnd.randint(1, 900)
        C1 = rnd.randint(1, S + 10)
        C2 = rnd.randint(1, S + 10)
        yield d, I, S, C1, C2, rnd.random() < 0.5


@pytest.mark.parametrize("d,I,S,C1,C2,with_res", list(_draws(12)))
def test_random_shape(cuda_device, d, I, S, C1, C2, with_res):
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, "cpu", bf)
    x = synth.hidden(S, d, "cpu", bf)
    res = synth.hidden(S, d, "cpu", bf, seed=synth.SEED_X + 1) if with_res else None
    G = lambda t: None if t is None else t.to(cuda_device)  # noqa: E731
    o1 = torch.empty((S, d), dtype=bf, device=cuda_device)
    o2 = torch.empty_like(o1)
    _mom.mlp_minseq_fwd(G(x), G(res), G(wg), G(wu), G(wd), o1, C1)
    _mom.mlp_minseq_fwd(G(x), G(res), G(wg), G(wu), G(wd), o2, C2)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    check_close(o1.cpu(), oracle.mlp_minseq(x, res, wg, wu, wd, C=C1), TOL_BF16, f"d={d} I={I} S={S} C={C1}")


def _gemv_draws(n, seed=321):
    rnd = random.Random(seed)
    for _ in range(n):
        d = 8 * rnd.randint(1, 640)     # 8 .. 5120
        I = 8 * rnd.randint(1, 2400)    # 8 .. 19200
        V = rnd.randint(1, 40000)
        yield d, I, V, rnd.random() < 0.5, rnd.choice([0.0, 1e-6, 1e-5, 0.5])


@pytest.mark.parametrize("d,I,V,with_res,eps", list(_gemv_draws(10)))
def test_random_shape_last_token_and_head(cuda_device, d, I, V, with_res, eps):
    """Random last-token shapes (any hidden / intermediate multiple of 8, any vocab): the GEMV pair, the
    folded-norm GEMV and the LM head + argmax against the oracle (argmax exact on the oracle's logits of
    the kernel's own hidden vector)."""
    from tests.parity import assert_argmax_exact
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, "cpu", bf)
    wh = synth.head_weight(V, d, "cpu", bf)
    gain = synth.norm_gain(d, "cpu", bf)
    x = synth.hidden(2, d, "cpu", bf)
    res = synth.hidden(2, d, "cpu", bf, seed=synth.SEED_X + 1) if with_res else None
    G = lambda t: None if t is None else t.to(cuda_device)  # noqa: E731
    y = torch.empty(d, dtype=bf, device=cuda_device)
    _mom.mlp_last_token(G(x)[1], None if res is None else G(res)[1], G(wg), G(wu), G(wd), y)
    logits = torch.empty(V, dtype=torch.float32, device=cuda_device)
    am = torch.empty(1, dtype=torch.int32, device=cuda_device)
    _mom.lm_head_last(y, G(gain), eps, G(wh), logits, am)
    yn_ = torch.empty(d, dtype=bf, device=cuda_device)
    wg_f, wu_f = _mom.fold_norm_gain(G(wg), G(gain)), _mom.fold_norm_gain(G(wu), G(gain))
    _mom.mlp_last_token_rmsnorm(G(x)[1], wg_f, wu_f, G(wd), yn_, 1e-5)
    torch.cuda.synchronize()
    regress = None if d >= 256 else 0
    check_close(y.cpu(), oracle.mlp_rows(x, res, wg, wu, wd, [1])[0], TOL_BF16, f"last token d={d} I={I}", regress)
    check_close(yn_.cpu(), oracle.mlp_norm_rows(x, gain, 1e-5, wg, wu, wd, [1])[0], TOL_BF16,
                f"last token rmsnorm d={d} I={I}", regress)
    ref = oracle.lm_head(oracle.rmsnorm(y.cpu().double().numpy(), gain, eps), wh)[0]
    check_close(logits.cpu(), ref, 1e-4, f"head d={d} V={V} eps={eps}")
    assert_argmax_exact(int(am.item()), ref, f"head d={d} V={V}")
