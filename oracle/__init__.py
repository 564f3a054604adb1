"""CPU oracle for the MOM mini-sequence prefill MLP path (arXiv 2504.12526).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The product package ``paper_2504_12526_b200`` never imports it, and the two share no
code: this wraps ``oracle/mom_oracle.c`` (plain C, float64 accumulation) via ctypes.

Every function follows a passage of PAPER.md (``P:<line>``) or SPEC.md (``S:<line>``):

* :func:`plan`          Alg. 1, M = ceil(S/C); sizes (C, ..., C, S-(M-1)C).
* :func:`mlp_minseq`    Alg. 1, O_i = MLP(A_i) for each mini-sequence, concat.
* :func:`mlp_rows`      the same MLP on a sampled list of rows (rows are independent).
* :func:`rmsnorm`       S:126 / S:270, the final norm before the head.
* :func:`lm_head`       Alg. 1, logits of the given rows.
* :func:`argmax_f32`    S:329, ties -> lowest index, decided in fp32 (the kernel's precision).

Pins for each of these live in ``tests/test_oracle.py`` (all ``-m "not gpu"``).
No parity is unpinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mom_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/mom_oracle.c with gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-pthread", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, p, i32, dbl = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        lib.oracle_plan.restype = i64
        lib.oracle_plan.argtypes = [i64, i64, p, p, i64]
        lib.oracle_mlp_rows.restype = i32
        lib.oracle_mlp_rows.argtypes = [p, p, p, p, p, p, i64, i64, i64, p, i32]
        lib.oracle_mlp_minseq.restype = i32
        lib.oracle_mlp_minseq.argtypes = [p, p, p, p, p, i64, i64, i64, i64, p, i32]
        lib.oracle_mlp_norm_rows.restype = i32
        lib.oracle_mlp_norm_rows.argtypes = [p, p, dbl, p, p, p, p, i64, i64, i64, p, i32]
        lib.oracle_rmsnorm.restype = i32
        lib.oracle_rmsnorm.argtypes = [p, p, dbl, i64, p]
        lib.oracle_lm_head.restype = i32
        lib.oracle_lm_head.argtypes = [p, p, i64, i64, i64, p, i32]
        lib.oracle_argmax_f32.restype = i64
        lib.oracle_argmax_f32.argtypes = [p, i64]
        lib.oracle_argmax_f64.restype = i64
        lib.oracle_argmax_f64.argtypes = [p, i64]
        _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _f32(a) -> np.ndarray:
    """Exact widening to float32 (bf16 -> f32 is exact).  Accepts numpy or torch."""
    if a is None:
        return None
    if hasattr(a, "detach"):  # torch tensor (CPU); bf16 has no numpy dtype
        a = a.detach().to("cpu").float().numpy()
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def plan(S: int, C: int):
    """Alg. 1: list of (start, length) of the M = ceil(S/C) mini-sequences."""
    lib = _load()
    cap = max(1, (S + C - 1) // C) if C >= 1 else 1
    starts = np.zeros(cap, np.int64)
    lens = np.zeros(cap, np.int64)
    M = lib.oracle_plan(S, C, _ptr(starts), _ptr(lens), cap)
    if M < 0:
        raise ValueError("invalid S/C")
    return [(int(starts[i]), int(lens[i])) for i in range(M)]


def mlp_minseq(x, residual, w_gate, w_up, w_down, C: int, nthreads: int | None = None) -> np.ndarray:
    """Alg. 1 P:109-113 on all S rows; returns O = concat(O_1..O_M) as float64 [S, d]."""
    lib = _load()
    x, residual = _f32(x), _f32(residual)
    wg, wu, wd = _f32(w_gate), _f32(w_up), _f32(w_down)
    S, d = x.shape
    I = wg.shape[0]
    assert wg.shape == (I, d) and wu.shape == (I, d) and wd.shape == (d, I)
    out = np.zeros((S, d), np.float64)
    rc = lib.oracle_mlp_minseq(_ptr(x), _ptr(residual), _ptr(wg), _ptr(wu), _ptr(wd),
                               S, d, I, C, _ptr(out), nthreads or default_threads())
    if rc != 0:
        raise RuntimeError("oracle_mlp_minseq failed")
    return out


def mlp_rows(x, residual, w_gate, w_up, w_down, rows, nthreads: int | None = None) -> np.ndarray:
    """The SwiGLU MLP on the listed rows: float64 [len(rows), d]."""
    lib = _load()
    x, residual = _f32(x), _f32(residual)
    wg, wu, wd = _f32(w_gate), _f32(w_up), _f32(w_down)
    S, d = x.shape
    I = wg.shape[0]
    assert wg.shape == (I, d) and wu.shape == (I, d) and wd.shape == (d, I)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    assert rows.ndim == 1 and (rows.size == 0 or (rows.min() >= 0 and rows.max() < S))
    out = np.zeros((rows.size, d), np.float64)
    rc = lib.oracle_mlp_rows(_ptr(x), _ptr(residual), _ptr(wg), _ptr(wu), _ptr(wd),
                             _ptr(rows), rows.size, d, I, _ptr(out), nthreads or default_threads())
    if rc != 0:
        raise RuntimeError("oracle_mlp_rows failed")
    return out


def mlp_norm_rows(x, gain, eps: float, w_gate, w_up, w_down, rows, nthreads: int | None = None) -> np.ndarray:
    """f3: out = x + MLP(RMSNorm(x) * gain) on the listed rows, float64 [len(rows), d]."""
    lib = _load()
    x, g = _f32(x), _f32(gain)
    wg, wu, wd = _f32(w_gate), _f32(w_up), _f32(w_down)
    S, d = x.shape
    I = wg.shape[0]
    assert g.shape == (d,) and wg.shape == (I, d) and wu.shape == (I, d) and wd.shape == (d, I)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((rows.size, d), np.float64)
    rc = lib.oracle_mlp_norm_rows(_ptr(x), _ptr(g), float(eps), _ptr(wg), _ptr(wu), _ptr(wd), _ptr(rows),
                                  rows.size, d, I, _ptr(out), nthreads or default_threads())
    if rc != 0:
        raise RuntimeError("oracle_mlp_norm_rows failed")
    return out


def rmsnorm(y, gain, eps: float) -> np.ndarray:
    """y / sqrt(mean(y^2) + eps) * gain (gain None = ones), one row, float64."""
    lib = _load()
    y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
    g = _f32(gain)
    out = np.zeros_like(y)
    rc = lib.oracle_rmsnorm(_ptr(y), _ptr(g), float(eps), y.size, _ptr(out))
    if rc != 0:
        raise RuntimeError("oracle_rmsnorm failed")
    return out


def lm_head(h, w_head, nthreads: int | None = None) -> np.ndarray:
    """Alg. 1: logits [n, V] = h [n, d] . W_head[V, d]^T, float64."""
    lib = _load()
    h = np.ascontiguousarray(h, dtype=np.float64)
    if h.ndim == 1:
        h = h.reshape(1, -1)
    w = _f32(w_head)
    n, d = h.shape
    V = w.shape[0]
    assert w.shape == (V, d)
    out = np.zeros((n, V), np.float64)
    rc = lib.oracle_lm_head(_ptr(h), _ptr(w), n, V, d, _ptr(out), nthreads or default_threads())
    if rc != 0:
        raise RuntimeError("oracle_lm_head failed")
    return out


def argmax_f32(logits) -> int:
    """S:329 greedy token: argmax of fp32 logits, ties -> lowest index."""
    lib = _load()
    a = _f32(logits).reshape(-1)
    return int(lib.oracle_argmax_f32(_ptr(a), a.size))


def argmax_f64(logits) -> int:
    lib = _load()
    a = np.ascontiguousarray(logits, dtype=np.float64).reshape(-1)
    return int(lib.oracle_argmax_f64(_ptr(a), a.size))


def last_token_logits(x, residual, w_gate, w_up, w_down, gain, eps, w_head):
    """Alg. 1, final-layer branch: A_last = A[-1], O_last = MLP(A_last)
    (P:103), L = LM_Head(rmsnorm(O_last)).  Returns (y_last, logits)."""
    x = _f32(x)
    S = x.shape[0]
    y = mlp_rows(x, residual, w_gate, w_up, w_down, [S - 1])[0]
    yn = rmsnorm(y, gain, eps) if gain is not None else y
    return y, lm_head(yn, w_head)[0]
