"""Comparators shared by the parity tests (test infrastructure, not product code).

Tolerances (BASELINE.json north_star):
  * bf16 MLP outputs: max relative error <= 2e-2, read normwise:
        err = max|gpu - ref| / max|ref|, per tensor AND per row.
  * fp32 variants: the same metric <= 1e-4.
  * last-token argmax: bit-exact (given the same hidden vector), with a tie guard:
    when the oracle's top-2 gap is below the fp32 accumulation bound the test reports a
    near-tie and accepts any index inside the bound instead of failing.
"""
from __future__ import annotations

import numpy as np

TOL_BF16 = 2e-2
TOL_F32 = 1e-4


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


def check_close(got, ref, tol: float, what: str = "") -> float:
    """Gate: normwise error per tensor and per row both <= tol.  Returns tensor error."""
    e = normwise_err(got, ref)
    r = rowwise_err(got, ref)
    worst = int(np.argmax(r)) if r.size else -1
    assert e <= tol and (r.size == 0 or r.max() <= tol), (
        f"{what}: normwise err {e:.3e}, worst row {worst} err {r.max() if r.size else 0:.3e} > tol {tol:.1e}")
    return e


def argmax_matches(gpu_idx: int, ref_logits, bound_rel: float = 1e-5) -> str:
    """Returns "exact" when gpu_idx equals the oracle argmax (ties -> lowest index) or
    "near-tie" when it differs but lies within the accumulation bound of the max.
    Raises AssertionError otherwise."""
    ref = as_f64(ref_logits).reshape(-1)
    best = int(np.argmax(ref))  # numpy argmax returns the first (lowest) index of the max
    if gpu_idx == best:
        return "exact"
    bound = bound_rel * np.max(np.abs(ref))
    assert 0 <= gpu_idx < ref.size and ref[best] - ref[gpu_idx] <= bound, (
        f"argmax {gpu_idx} != oracle {best} (gap {ref[best] - ref[gpu_idx]:.3e} > {bound:.3e})")
    return "near-tie"
