"""Edge cases of the tcgen05 path: K tails (hidden not a multiple of the 64-wide K stage),
N tails in both phases, a single token (S = 1), mini-sequences of one row, and the memory claim
of Eq. 1 / Eq. 3: the MLP's transient device memory is one mini-sequence's
C * I * w bytes, i.e. M times less than the unchunked S * I * w."""
from __future__ import annotations

import pytest
import torch

import oracle
import synth
from paper_2504_12526_b200 import _mom
from tests.parity import TOL_BF16, check_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("S,d,I,C", [(333, 200, 328, 100),   # K tail 8 of 64 (phase A), N tails both phases
                                     (1, 256, 512, 1),       # one token
                                     (5, 264, 136, 2),       # tiny, ragged everything
                                     (260, 1032, 2056, 257)])  # 1032 = 16*64 + 8, 2056 = 16*128 + 8
def test_tails_vs_oracle(cuda_device, S, d, I, C):
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, "cpu", bf)
    x = synth.hidden(S, d, "cpu", bf)
    res = synth.hidden(S, d, "cpu", bf, seed=synth.SEED_X + 1)
    out = torch.empty((S, d), dtype=bf, device=cuda_device)
    _mom.mlp_minseq_fwd(x.to(cuda_device), res.to(cuda_device), wg.to(cuda_device), wu.to(cuda_device),
                        wd.to(cuda_device), out, C)
    torch.cuda.synchronize()
    check_close(out.cpu(), oracle.mlp_minseq(x, res, wg, wu, wd, C=C), TOL_BF16, f"S={S} d={d} I={I} C={C}")


def test_transient_memory_is_one_minisequence(cuda_device):
    """Peak extra device memory of the call = its workspace: C*I*w (+ a few hundred bytes of
    counters) at C = S/M, against S*I*w at C = S -- M-fold (SPEC S:505 acceptance idea)."""
    S, d, I, M = 16384, 1024, 3584, 8
    C = S // M
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    x = synth.hidden(S, d, cuda_device, bf)
    out = torch.empty_like(x)
    peaks = {}
    for c in (C, S):
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, c)  # the binding allocates the workspace
        torch.cuda.synchronize()
        peaks[c] = torch.cuda.max_memory_allocated() - base
    assert C * I * 2 <= peaks[C] <= C * I * 2 + (1 << 20)
    assert S * I * 2 <= peaks[S] <= S * I * 2 + (1 << 20)
    ratio = peaks[S] / peaks[C]
    assert M * 0.99 <= ratio <= M * 1.01


def test_concurrent_calls_from_two_threads(cuda_device):
    """include/mom.h claims thread safety: two host threads issuing calls on their own streams (own
    workspaces) at the same time get exactly the single-threaded results."""
    import threading
    S, d, I, C = 1200, 512, 1024, 300
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    xs = [synth.hidden(S, d, cuda_device, bf, seed=synth.SEED_X + k) for k in range(2)]
    refs = []
    for x in xs:
        o = torch.empty_like(x)
        _mom.mlp_minseq_fwd(x, x, wg, wu, wd, o, C)
        refs.append(o)
    torch.cuda.synchronize()
    outs = [torch.empty_like(x) for x in xs]
    errors = []

    def work(k):
        try:
            s = torch.cuda.Stream(cuda_device)
            with torch.cuda.stream(s):
                for _ in range(5):
                    _mom.mlp_minseq_fwd(xs[k], xs[k], wg, wu, wd, outs[k], C, stream=s)
            s.synchronize()
        except Exception as e:  # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for k in range(2):
        assert torch.equal(outs[k], refs[k])
