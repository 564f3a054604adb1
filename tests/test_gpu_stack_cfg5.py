"""BASELINE config 5 shapes on one GPU: Llama-3-8B MLP at S = 455000 tokens (M = 56 mini-sequences of
C = 8192, tail 4440 rows), KV [S, 2*1024] bf16 (1.86 GB per layer) offloaded and reloaded.  The stack is
cut to 4 layers (3 mini-sequence layers + last token) to bound test time; every per-layer step is the
same as at 32 layers.  Teacher-forced per-layer parity on sampled rows (random, boundaries, tail)."""
from __future__ import annotations

import pytest

import synth
from tests.test_gpu_stack import _run_stack

pytestmark = pytest.mark.gpu


def test_stack_cfg5_llama_455k_tokens(cuda_device):
    import psutil
    w = synth.CONFIGS[4]
    L = 4
    need = L * w.S * 2 * w.d_kv * 2
    if psutil.virtual_memory().available < 2 * need:
        pytest.skip(f"host has {psutil.virtual_memory().available / 1e9:.0f} GB free, needs {2 * need / 1e9:.0f} GB")
    assert -(-w.S // w.C) == 56 and w.S - 55 * w.C == 4440
    _run_stack(cuda_device, w.hidden, w.intermediate, w.vocab, L, w.S, w.C, w.d_kv, w.eps,
               check_layers=[0, L - 2], n_rows=8)
