"""The single-launch fused mini-sequence kernel (phase-B tiles wait on per-row-block counters
released by phase-A epilogues) must give exactly the bits of the two-launch path, for ragged
mini-sequences, both CTA-group variants, with and without residual and with the folded norm."""
from __future__ import annotations

import os

import pytest
import torch

import oracle
import synth
from paper_2504_12526_b200 import _mom
from tests.parity import TOL_BF16, check_close

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _env():
    keys = ("MOM_FUSED", "MOM_CTA_GROUP", "MOM_GROUP_M_A")
    old = {k: os.environ.get(k) for k in keys}
    yield
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _run(x, res, wg, wu, wd, C, fused, cg, group=None):
    os.environ["MOM_FUSED"] = "1" if fused else "0"
    os.environ["MOM_CTA_GROUP"] = cg
    if group is None:
        os.environ.pop("MOM_GROUP_M_A", None)
    else:
        os.environ["MOM_GROUP_M_A"] = str(group)
    out = torch.empty_like(x)
    _mom.mlp_minseq_fwd(x, res, wg, wu, wd, out, C)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("cg", ["1", "2"])
@pytest.mark.parametrize("S,d,I,C,group", [(1000, 256, 688, 300, None), (2000, 512, 1024, 1500, 1),
                                           (4096, 384, 640, 4096, 3), (77, 256, 384, 64, None)])
def test_fused_equals_two_launch(cuda_device, cg, S, d, I, C, group):
    bf = torch.bfloat16
    wg, wu, wd = (t.to(cuda_device) for t in synth.mlp_weights(d, I, 0, "cpu", bf))
    x = synth.hidden(S, d, cuda_device, bf)
    res = synth.hidden(S, d, cuda_device, bf, seed=synth.SEED_X + 1)
    a = _run(x, res, wg, wu, wd, C, False, cg)
    b = _run(x, res, wg, wu, wd, C, True, cg, group)
    assert torch.equal(a, b)
    c = _run(x, None, wg, wu, wd, C, True, cg, group)
    rows = list(range(0, S, max(1, S // 97))) + [S - 1]
    ref = oracle.mlp_rows(x.cpu(), None, wg.cpu(), wu.cpu(), wd.cpu(), rows)
    check_close(c[rows].cpu(), ref, TOL_BF16, "fused, no residual")


def test_fused_full_size_cfg2_repeatable(cuda_device):
    """Config 2 at full size: fused == two-launch bitwise, and repeated fused runs are identical
    (the counter protocol has no race that could let a phase-B tile read stale H)."""
    w = synth.CONFIGS[1]
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(w.hidden, w.intermediate, 0, cuda_device, bf)
    x = synth.hidden(w.S, w.hidden, cuda_device, bf)
    ref = _run(x, x, wg, wu, wd, w.C, False, "2")
    for _ in range(3):
        assert torch.equal(_run(x, x, wg, wu, wd, w.C, True, "2"), ref)
