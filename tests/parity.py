"""Comparators shared by the parity tests (test infrastructure, not product code).

Tolerances (BASELINE.json north_star):
  * bf16 MLP outputs: max relative error <= 2e-2, read normwise:
        err = max|gpu - ref| / max|ref|, per tensor AND per row.
  * fp32 variants: the same metric <= 1e-4.
  * bf16 regression bound (beside the 2e-2 gate): the tensor-level
    normwise error must also stay <= REG_BF16 = 6e-3 at hidden >= 256.  Derivation: both sides
    get the same bf16 inputs; the kernel rounds H_i once and each output once (RNE, relative
    error <= 2^-9 = 1.95e-3 each) and accumulates in fp32 (K * 2^-24 ~ 1e-3 worst case at
    K = 14336, ~1e-5 typical); the H rounding errors enter the down GEMM with random signs, so
    they add ~2^-9/sqrt(3) of the row norm per output, a few sigma at the max.  6e-3 ~ 3 x 2^-9
    is the sum of those terms with margin; a systematic error (a dropped K slice at d = 4096
    removes 1/64 of the sum, ~1.6e-2) fails it while passing the 2e-2 gate.
  * last-token argmax: bit-exact against the float64 oracle's argmax (given the same hidden
    vector); every comparison logs the oracle's top-2 gap so a failure can be read as a near
    tie or a real error.  Each gated comparison is recorded in RECORDS and printed in the
    pytest terminal summary (tests/conftest.py).
"""
from __future__ import annotations

import numpy as np

TOL_BF16 = 2e-2
TOL_F32 = 1e-4
REG_BF16 = 6e-3

# (kind, what, value, limit) of every comparison of this session; printed by conftest
RECORDS: list = []


def as_f64(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().to("cpu").double().numpy()
    return np.asarray(a, dtype=np.float64)


def normwise_err(got, ref) -> float:
    got, ref = as_f64(got), as_f64(ref)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    if not np.all(np.isfinite(got)):
        return float("inf")
    denom = np.max(np.abs(ref))
    num = np.max(np.abs(got - ref)) if got.size else 0.0
    if denom == 0.0:
        return float(num)
    return float(num / denom)


def rowwise_err(got, ref) -> np.ndarray:
    got, ref = as_f64(got), as_f64(ref)
    if got.ndim == 1:
        got, ref = got[None], ref[None]
    denom = np.max(np.abs(ref), axis=1)
    denom = np.where(denom == 0.0, 1.0, denom)
    return np.max(np.abs(got - ref), axis=1) / denom


def check_close(got, ref, tol: float, what: str = "", regress: float | None = None) -> float:
    """Gate: normwise error per tensor and per row both <= tol.  For bf16 (tol == TOL_BF16) with a
    row length >= 256 the tensor error must also be <= REG_BF16 (pass regress=0 to skip, e.g. for
    outputs that are not a single rounding of an fp32-accumulated value).  Returns tensor error."""
    e = normwise_err(got, ref)
    r = rowwise_err(got, ref)
    worst = int(np.argmax(r)) if r.size else -1
    if regress is None:
        n = as_f64(ref).shape[-1] if as_f64(ref).ndim else 1
        regress = REG_BF16 if (tol == TOL_BF16 and n >= 256) else 0
    RECORDS.append(("close", what, e, float(r.max()) if r.size else 0.0, tol, regress))
    assert e <= tol and (r.size == 0 or r.max() <= tol), (
        f"{what}: normwise err {e:.3e}, worst row {worst} err {r.max() if r.size else 0:.3e} > tol {tol:.1e}")
    assert not regress or e <= regress, f"{what}: normwise err {e:.3e} > regression bound {regress:.1e}"
    return e


def top2_gap(ref_logits) -> tuple[int, float, float]:
    """(argmax with ties -> lowest index, top-1 minus top-2 logit, that gap / max|logit|)."""
    ref = as_f64(ref_logits).reshape(-1)
    best = int(np.argmax(ref))  # numpy argmax returns the first (lowest) index of the max
    if ref.size < 2:
        return best, float("inf"), float("inf")
    rest = np.delete(ref, best)
    gap = float(ref[best] - rest.max())
    return best, gap, gap / max(float(np.max(np.abs(ref))), 1e-300)


def assert_argmax_exact(gpu_idx: int, ref_logits, what: str = "") -> float:
    """Bit-exact argmax against the float64 oracle's logits; records and returns the
    oracle's relative top-2 gap (the margin the kernel's fp32 accumulation had to respect)."""
    best, gap, rel = top2_gap(ref_logits)
    RECORDS.append(("argmax", what, float(rel), float(gap), gpu_idx, best))
    assert gpu_idx == best, (f"{what}: argmax {gpu_idx} != oracle {best} (oracle top-2 gap {gap:.3e}, "
                             f"{rel:.2e} of max|logit|)")
    return rel
