"""BASELINE config 5 on one GPU: Llama-3-8B MLP at S = 455000 tokens (M = 56 mini-sequences of C = 8192,
tail 4440 rows), KV [S, 2*1024] bf16 (1.86 GB per layer) offloaded and reloaded.  All 32 layers (31
mini-sequence layers + the last token) with the budgeted early reload (f4) when the host can pin the
59.6 GB of offloaded K/V, else the first 4 layers.  Teacher-forced per-layer parity on sampled rows
(random, boundaries, tail), last-token MLP, LM head, exact argmax, offloaded/reloaded bytes."""
from __future__ import annotations

import pytest

import synth
from tests.test_gpu_stack import _run_stack

pytestmark = pytest.mark.gpu


def test_stack_cfg5_llama_455k_tokens(cuda_device):
    import psutil
    w = synth.CONFIGS[4]
    per_layer = w.S * 2 * w.d_kv * 2
    L = w.layers if psutil.virtual_memory().available >= 1.5 * w.layers * per_layer else 4
    if psutil.virtual_memory().available < 2 * L * per_layer and L == 4:
        pytest.skip(f"host has {psutil.virtual_memory().available / 1e9:.0f} GB free")
    assert -(-w.S // w.C) == 56 and w.S - 55 * w.C == 4440
    checks = [0, L // 2, L - 2] if L > 4 else [0, L - 2]
    _run_stack(cuda_device, w.hidden, w.intermediate, w.vocab, L, w.S, w.C, w.d_kv, w.eps,
               check_layers=checks, n_rows=8, early="auto")
