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
