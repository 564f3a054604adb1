"""Pins for the CPU oracle (oracle/), all CPU-only (-m "not gpu").

Each test ties an oracle function to something other than itself: the worked values
printed in SPEC.md (tests/golden/spec_worked_examples.json, each with its citation),
closed forms of special cases, an exact high-precision brute force on tiny inputs, and
the two facts the paper fixes (sec. 4.5 "output logits ... were identical"):
F1 bit-identity for every mini-sequence count M, F2 last-token head == last row of the
full head.  The one-hot tests are built so that a transposed operand, swapped gate/up,
a dropped term or a sign error in the sigmoid fails at least one of them.
"""
from __future__ import annotations

import json
import math
import os
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.parity import TOL_BF16, check_close, normwise_err

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def rng_f32(shape, seed, scale=1.0):
    r = np.random.default_rng(seed)
    return (r.standard_normal(shape) * scale).astype(np.float32)


# ------------------------------------------------------------------ a1: partition plan
def test_plan_worked_examples():
    g = GOLD["partition_8_3"]
    assert [n for _, n in oracle.plan(g["S"], g["C"])] == g["expect_sizes"]
    assert [s for s, _ in oracle.plan(8, 3)] == [0, 3, 6]
    g = GOLD["partition_c_ge_s"]
    assert len(oracle.plan(g["S"], g["C"])) == g["expect_M"]
    g = GOLD["partition_144000"]
    assert len(oracle.plan(g["S"], g["C"])) == g["expect_M"]
    # SURVEY §8(a) a1 tails: 155000 / 8192 -> 19, last 7544
    p = oracle.plan(155000, 8192)
    assert len(p) == 19 and p[-1][1] == 7544


@pytest.mark.parametrize("S,C", [(1, 1), (7, 2), (1024, 256), (1000, 7), (65536, 8192), (5, 100)])
def test_plan_is_a_partition(S, C):
    p = oracle.plan(S, C)
    assert len(p) == math.ceil(S / C)
    pos = 0
    for i, (s, n) in enumerate(p):
        assert s == pos and 1 <= n <= C
        if i < len(p) - 1:
            assert n == C
        pos += n
    assert pos == S


# ------------------------------------------------------------------ a2/a3: SwiGLU MLP
def _mlp1(x, wg, wu, wd, res=None):
    x = np.asarray(x, np.float32).reshape(1, -1)
    r = None if res is None else np.asarray(res, np.float32).reshape(1, -1)
    return oracle.mlp_rows(x, r, np.asarray(wg, np.float32), np.asarray(wu, np.float32),
                           np.asarray(wd, np.float32), [0])[0]


def test_swiglu_spec_worked_values():
    g = GOLD["swiglu_ones"]
    out = _mlp1([1.0], [[1.0]], [[1.0]], [[1.0]])
    assert abs(out[0] - g["expect"]) < g["abs_tol"]
    assert _mlp1([0.0], [[1.0]], [[1.0]], [[1.0]])[0] == GOLD["swiglu_zero"]["expect"]
    # x = 0 with a residual -> the residual exactly
    assert _mlp1([0.0], [[1.0]], [[1.0]], [[1.0]], res=[0.375])[0] == 0.375


def test_swiglu_one_hot_structure():
    """d=2, I=3 one-hot weights with x = [0.5, 2].  sigma(2) = 0.8807970779778823.
    Case A: Wg[2,1] = Wu[2,1] = 1, Wd[0,2] = 1  ->  out = [2*sigma(2)*2, 0] = [4 sigma(2), 0].
    Case B: Wg[0,1] = 1 (gate reads x_1 = 2), Wu[0,0] = 1 (up reads x_0 = 0.5), Wd[1,0] = 1
            -> out = [0, swish(2) * 0.5] = [0, sigma(2)].  Swapping gate and up would give
            swish(0.5) * 2 = sigma(0.5) = 0.6225, transposing any weight breaks the shapes
            or moves the hot element."""
    s2 = 0.8807970779778823
    x = [0.5, 2.0]
    wg = np.zeros((3, 2)); wu = np.zeros((3, 2)); wd = np.zeros((2, 3))
    wg[2, 1] = wu[2, 1] = 1.0; wd[0, 2] = 1.0
    out = _mlp1(x, wg, wu, wd)
    assert abs(out[0] - 4 * s2) < 1e-14 and out[1] == 0.0
    wg = np.zeros((3, 2)); wu = np.zeros((3, 2)); wd = np.zeros((2, 3))
    wg[0, 1] = 1.0; wu[0, 0] = 1.0; wd[1, 0] = 1.0
    out = _mlp1(x, wg, wu, wd)
    assert out[0] == 0.0 and abs(out[1] - s2) < 1e-14


def test_swiglu_closed_form_identity_weights():
    """d = I, Wg = Wu = Wd = identity, residual = x  ->  out = x + x * swish(x) = x + x^2 sigma(x)."""
    d = 8
    x = rng_f32((4, d), 1)
    eye = np.eye(d, dtype=np.float32)
    out = oracle.mlp_minseq(x, x, eye, eye, eye, C=3)
    xd = x.astype(np.float64)
    expect = xd + xd * xd / (1.0 + np.exp(-xd))
    assert np.max(np.abs(out - expect)) < 1e-14


def test_swiglu_odd_part():
    """d = I = 1, all weights 1: out(x) = x * swish(x); out(x) + out(-x) = x (swish(x) - swish(-x)) = x^2."""
    for xv in [0.25, 1.0, 3.0, 7.5]:
        a = _mlp1([xv], [[1.0]], [[1.0]], [[1.0]])[0]
        b = _mlp1([-xv], [[1.0]], [[1.0]], [[1.0]])[0]
        assert abs((a + b) - xv * xv) < 1e-13 * max(1.0, xv * xv)


def test_swiglu_zero_up_gives_residual_exactly():
    d, I = 16, 24
    x = rng_f32((5, d), 2)
    res = rng_f32((5, d), 3)
    wg = rng_f32((I, d), 4)
    wd = rng_f32((d, I), 5)
    out = oracle.mlp_minseq(x, res, wg, np.zeros((I, d), np.float32), wd, C=2)
    assert np.array_equal(out, res.astype(np.float64))


def _exact_mlp_row(x, wg, wu, wd, res=None):
    """Brute force in exact rationals (projections) + 60-digit Decimal (exp)."""
    getcontext().prec = 60
    d = len(x)
    I = wg.shape[0]
    X = [Fraction(float(v)) for v in x]
    h = []
    for j in range(I):
        g = sum((X[k] * Fraction(float(wg[j, k])) for k in range(d)), Fraction(0))
        u = sum((X[k] * Fraction(float(wu[j, k])) for k in range(d)), Fraction(0))
        gd = Decimal(g.numerator) / Decimal(g.denominator)
        ud = Decimal(u.numerator) / Decimal(u.denominator)
        h.append(gd / (Decimal(1) + (-gd).exp()) * ud)
    out = []
    for c in range(wd.shape[0]):
        o = sum((h[j] * Decimal(float(wd[c, j])) for j in range(I)), Decimal(0))
        if res is not None:
            o += Decimal(float(res[c]))
        out.append(float(o))
    return np.array(out)


def test_swiglu_exact_brute_force():
    """Oracle float64 vs an exact evaluation: error within the float64 accumulation bound."""
    S, d, I = 3, 6, 10
    x = rng_f32((S, d), 10)
    res = rng_f32((S, d), 11)
    wg, wu, wd = rng_f32((I, d), 12, 0.5), rng_f32((I, d), 13, 0.5), rng_f32((d, I), 14, 0.3)
    out = oracle.mlp_minseq(x, res, wg, wu, wd, C=2)
    for r in range(S):
        ex = _exact_mlp_row(x[r], wg, wu, wd, res[r])
        assert np.max(np.abs(out[r] - ex)) <= 1e-13 * max(1.0, np.max(np.abs(ex)))


# ------------------------------------------------------------------ F1: bit-identity across M
@pytest.mark.parametrize("S", [1, 2, 7, 8, 257])
def test_F1_bit_identical_for_every_M(S):
    """P:286 (logits identical) via P:109-113 (row partition of a position-wise op)."""
    d, I = 12, 20
    x = rng_f32((S, d), 20 + S)
    res = rng_f32((S, d), 40 + S)
    wg, wu, wd = rng_f32((I, d), 21, 0.3), rng_f32((I, d), 22, 0.3), rng_f32((d, I), 23, 0.2)
    ref = oracle.mlp_minseq(x, res, wg, wu, wd, C=S)
    for C in sorted({1, 3, 16, 64, max(1, S - 1), S, S + 3}):
        for nt in (1, 3):
            out = oracle.mlp_minseq(x, res, wg, wu, wd, C=C, nthreads=nt)
            assert out.tobytes() == ref.tobytes(), (S, C, nt)
    rows = list(range(S))[::-1]
    sampled = oracle.mlp_rows(x, res, wg, wu, wd, rows)
    assert sampled.tobytes() == ref[rows].tobytes()


def test_F1_detects_single_bit_flip():
    """the equivalence comparator must fail when one weight bit is flipped."""
    S, d, I = 9, 8, 12
    x = rng_f32((S, d), 60)
    wg, wu, wd = rng_f32((I, d), 61), rng_f32((I, d), 62), rng_f32((d, I), 63)
    ref = oracle.mlp_minseq(x, None, wg, wu, wd, C=4)
    wd2 = wd.copy()
    wd2.view(np.uint32)[3, 5] ^= np.uint32(1)  # lowest mantissa bit of one weight
    out = oracle.mlp_minseq(x, None, wg, wu, wd2, C=4)
    assert out.tobytes() != ref.tobytes()
    wd3 = wd.copy()
    wd3.view(np.uint32)[3, 5] ^= np.uint32(1 << 29)  # an exponent bit: the tolerance gate fails too
    out3 = oracle.mlp_minseq(x, None, wg, wu, wd3, C=4)
    with pytest.raises(AssertionError):
        check_close(out3, ref, TOL_BF16, "mutated")


# ------------------------------------------------------------------ a7: RMSNorm + LM head
def test_rmsnorm_spec_worked_values():
    g = GOLD["rmsnorm_34"]
    out = oracle.rmsnorm(np.array(g["x"], float), np.array(g["gain"], np.float32), g["eps"])
    assert np.max(np.abs(out - np.array(g["expect"]))) < g["abs_tol"]
    g = GOLD["rmsnorm_const"]
    assert np.array_equal(oracle.rmsnorm(np.array(g["x"], float), None, g["eps"]), np.array(g["expect"], float))
    g = GOLD["rmsnorm_zero"]
    assert np.array_equal(oracle.rmsnorm(np.array(g["x"], float), None, g["eps"]), np.array(g["expect"], float))
    # eps placement (eps inside the square root), with eps large enough that every other
    # placement (outside the root, added to the rms, dropped) gives a different value
    g = GOLD["rmsnorm_eps_inside"]
    out = oracle.rmsnorm(np.array(g["x"], float), np.array(g["gain"], np.float32), g["eps"])
    assert np.array_equal(out, np.array(g["expect"], float))
    g = GOLD["rmsnorm_eps_34"]
    out = oracle.rmsnorm(np.array(g["x"], float), None, g["eps"])
    assert np.max(np.abs(out - np.array(g["expect"]))) < g["abs_tol"]
    # gain scales elementwise: [3,4] with gain [2, -1]
    out = oracle.rmsnorm(np.array([3.0, 4.0]), np.array([2.0, -1.0], np.float32), 0.0)
    assert np.max(np.abs(out - np.array([2 * 0.84852814, -1.13137085]))) < 1e-8


def test_lm_head_spec_matmul():
    """S:121 [[1,2],[3,4]] . [[5,6],[7,8]] = [[19,22],[43,50]].  W_head is [V, d]
    (nn.Linear), so W_head = B^T = [[5,7],[6,8]]."""
    g = GOLD["matmul"]
    a = np.array(g["a"], float)
    w = np.array(g["b"], np.float32).T.copy()
    assert np.array_equal(oracle.lm_head(a, w), np.array(g["expect"], float))


def test_lm_head_identity_padded():
    g = GOLD["lm_head_identity"]
    V, d, hot = g["V"], g["d"], g["hot"]
    w = np.zeros((V, d), np.float32)
    for i in range(min(V, d)):
        w[i, i] = 1.0
    e = np.zeros(d); e[hot] = 1.0
    expect = np.zeros(V); expect[hot] = 1.0
    assert np.array_equal(oracle.lm_head(e, w)[0], expect)


def test_argmax_spec_and_ties():
    g = GOLD["argmax_unique"]
    lg = np.zeros(g["logits_len"], np.float32); lg[g["max_at"]] = 1.0
    assert oracle.argmax_f32(lg) == g["expect"]
    g = GOLD["argmax_tie"]
    lg = np.zeros(g["logits_len"], np.float32); lg[g["max_at"]] = 3.0
    assert oracle.argmax_f32(lg) == g["expect"] and oracle.argmax_f64(lg.astype(float)) == g["expect"]
    lg = -np.abs(rng_f32(1000, 70)) - 1.0  # all negative, max somewhere
    assert oracle.argmax_f32(lg) == int(np.argmax(lg))


def test_F2_last_token_head_equals_last_row_of_full_head():
    """P:102-105 vs the standard path; P:286 identical logits."""
    S, d, I, V = 33, 16, 40, 50
    x = rng_f32((S, d), 80)
    res = rng_f32((S, d), 81)
    wg, wu, wd = rng_f32((I, d), 82, 0.3), rng_f32((I, d), 83, 0.3), rng_f32((d, I), 84, 0.2)
    wh = rng_f32((V, d), 85, 0.25)
    gain = (1 + 0.1 * rng_f32(d, 86)).astype(np.float32)
    # standard path: MLP on every row, norm every row, head on every row
    full = oracle.mlp_minseq(x, res, wg, wu, wd, C=S)
    normed = np.stack([oracle.rmsnorm(full[r], gain, 1e-5) for r in range(S)])
    logits_full = oracle.lm_head(normed, wh)
    # MOM path: last token only (Alg. 1 final branch)
    y, logits_last = oracle.last_token_logits(x, res, wg, wu, wd, gain, 1e-5, wh)
    assert y.tobytes() == full[S - 1].tobytes()
    assert logits_last.tobytes() == logits_full[S - 1].tobytes()
    assert oracle.argmax_f64(logits_last) == oracle.argmax_f64(logits_full[S - 1])


# ------------------------------------------------------------------ Eq. 1-3 accounting
def test_memory_formulas_spec_values():
    """Eq. 1 intermediate S*I*w; Eq. 3 S*I*w/M; Eq. 2 KV 2*S*d*L*w."""
    g = GOLD["eq1_bytes"]
    assert g["S"] * g["I"] * g["w"] == g["expect"]
    g = GOLD["eq3_bytes"]
    C = math.ceil(g["S"] / g["M"])
    assert C * g["I"] * g["w"] == g["expect"]  # one mini-sequence's intermediate
    for key in ("kv_bytes", "kv_reload_bytes"):
        g = GOLD[key]
        assert 2 * g["S"] * g["d"] * g["L"] * g["w"] == g["expect"]


def test_normwise_comparator():
    ref = np.array([[1.0, -2.0], [0.5, 4.0]])
    assert normwise_err(ref, ref) == 0.0
    got = ref.copy(); got[1, 1] += 0.04
    assert abs(normwise_err(got, ref) - 0.01) < 1e-15
    assert normwise_err(np.array([np.nan]), np.array([1.0])) == float("inf")


# ------------------------------------------------------------------ f3: norm folded into the MLP
def test_norm_block_unit_rms_equals_plain_mlp():
    """rows of +-1 have mean(x^2) = 1 exactly: with gain 1 and eps 0 RMSNorm is the identity, so the
    block equals x + MLP(x) bitwise."""
    S, d, I = 6, 16, 24
    r = np.random.default_rng(90)
    x = np.where(r.random((S, d)) < 0.5, -1.0, 1.0).astype(np.float32)
    wg, wu, wd = rng_f32((I, d), 91, 0.3), rng_f32((I, d), 92, 0.3), rng_f32((d, I), 93, 0.2)
    out = oracle.mlp_norm_rows(x, np.ones(d, np.float32), 0.0, wg, wu, wd, list(range(S)))
    ref = oracle.mlp_rows(x, x, wg, wu, wd, list(range(S)))
    assert out.tobytes() == ref.tobytes()


SIGMA_HALF = 0.6224593312018546  # sigma(0.5) = 1 / (1 + e^-0.5), textbook value
SIGMA_ONE = 0.7310585786300049   # sigma(1)


def test_norm_block_eps_placement():
    """S:126 eps inside the root, pinned through the f3 block (S:260 x + MLP(RMSNorm(x) * g)).
    d = I = 2, identity weights, so out_c = x_c + xn_c * swish(xn_c) = x_c + xn_c^2 sigma(xn_c).
    x = [1, 1], eps = 3 -> xn = [0.5, 0.5] (1/sqrt(1+3)); eps outside the root would give 0.25."""
    eye = np.eye(2, dtype=np.float32)
    x = np.array([[1.0, 1.0]], np.float32)
    out = oracle.mlp_norm_rows(x, np.ones(2, np.float32), 3.0, eye, eye, eye, [0])[0]
    assert np.max(np.abs(out - (1.0 + 0.25 * SIGMA_HALF))) < 1e-15
    # gain 2 doubles xn to 1.0: out = 1 + sigma(1)
    out = oracle.mlp_norm_rows(x, np.full(2, 2.0, np.float32), 3.0, eye, eye, eye, [0])[0]
    assert np.max(np.abs(out - (1.0 + SIGMA_ONE))) < 1e-15
    # eps = 0 on the same row: xn = x = 1 -> 1 + sigma(1)
    out = oracle.mlp_norm_rows(x, np.ones(2, np.float32), 0.0, eye, eye, eye, [0])[0]
    assert np.max(np.abs(out - (1.0 + SIGMA_ONE))) < 1e-15


def test_norm_block_closed_forms():
    S, d, I = 5, 12, 20
    x = rng_f32((S, d), 94, 3.0)
    wg, wu, wd = rng_f32((I, d), 95, 0.3), rng_f32((I, d), 96, 0.3), rng_f32((d, I), 97, 0.2)
    rows = list(range(S))
    gain = (1 + 0.2 * rng_f32(d, 98)).astype(np.float32)
    # gain 0 -> normed input 0 -> MLP(0) = 0 -> out = x exactly
    assert np.array_equal(oracle.mlp_norm_rows(x, np.zeros(d, np.float32), 1e-6, wg, wu, wd, rows), x.astype(float))
    # RMSNorm is scale invariant (eps = 0): the MLP part of 2x equals that of x
    a = oracle.mlp_norm_rows(x, gain, 0.0, wg, wu, wd, rows) - x
    b = oracle.mlp_norm_rows(2 * x, gain, 0.0, wg, wu, wd, rows) - 2 * x.astype(float)
    assert np.max(np.abs(a - b)) <= 1e-13 * max(1.0, np.max(np.abs(a)))
    # composition: rmsnorm() then the plain MLP on the (float32-rounded) normed rows
    xn = np.stack([oracle.rmsnorm(x[i].astype(float), gain, 1e-5) for i in rows]).astype(np.float32)
    ref = oracle.mlp_rows(xn, x, wg, wu, wd, rows)
    got = oracle.mlp_norm_rows(x, gain, 1e-5, wg, wu, wd, rows)
    assert np.max(np.abs(got - ref)) <= 1e-6 * np.max(np.abs(ref))


# ------------------------------------------------------------------ F1, property-based
try:
    from hypothesis import given, settings, strategies as st
except ImportError:  # pragma: no cover
    given = None

if given is not None:
    @settings(max_examples=40, deadline=None)
    @given(S=st.integers(1, 40), C=st.integers(1, 50), d=st.integers(1, 9), I=st.integers(1, 11),
           seed=st.integers(0, 10_000), residual=st.booleans())
    def test_F1_property_any_partition(S, C, d, I, seed, residual):
        """P:109-113 / P:286 for random shapes and partitions: mini-sequence output == unchunked output
        bitwise, and any row subset (mlp_rows) equals the same rows of the full result bitwise."""
        x = rng_f32((S, d), seed)
        res = rng_f32((S, d), seed + 1) if residual else None
        wg, wu, wd = rng_f32((I, d), seed + 2, 0.5), rng_f32((I, d), seed + 3, 0.5), rng_f32((d, I), seed + 4, 0.5)
        ref = oracle.mlp_minseq(x, res, wg, wu, wd, C=S)
        assert oracle.mlp_minseq(x, res, wg, wu, wd, C=C).tobytes() == ref.tobytes()
        rows = sorted({(seed * 7 + k * 13) % S for k in range(min(S, 5))})
        assert oracle.mlp_rows(x, res, wg, wu, wd, rows).tobytes() == ref[rows].tobytes()
