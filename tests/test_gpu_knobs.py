"""The tuning knobs of include/mom.h change scheduling, caching and store paths only: every setting
must give the bitwise-identical output (and the same as the default)."""
from __future__ import annotations

import os

import pytest
import torch

import synth
from paper_2504_12526_b200 import _mom

pytestmark = pytest.mark.gpu

KNOBS = [{}, {"MOM_CTA_GROUP": "1"}, {"MOM_GROUP_M_A": "1"}, {"MOM_GROUP_M_A": "5", "MOM_GROUP_M_B": "3"},
         {"MOM_TMA_POLICY": "1"}, {"MOM_TMA_POLICY": "3"}, {"MOM_TMA_POLICY": "5"}, {"MOM_FUSED": "1"},
         {"MOM_FUSED": "1", "MOM_GROUP_M_A": "2"}, {"MOM_EPI_A_COALESCED": "0"}, {"MOM_NB_B": "256"},
         {"MOM_NB_B": "224"}, {"MOM_NB_B": "160"}, {"MOM_NB_B": "128"}, {"MOM_NB_B": "96"},
         {"MOM_NB_B": "224", "MOM_CTA_GROUP": "1"}, {"MOM_NB_B": "192", "MOM_FUSED": "1"}, {"MOM_MLP_PDL": "0"},
         {"MOM_MLP_PDL": "0", "MOM_CTA_GROUP": "1"}, {"MOM_HALF_TAIL": "0"}, {"MOM_HALF_TAIL": "0", "MOM_CTA_GROUP": "1"},
         {"MOM_EPI_L2_HINT": "0"}, {"MOM_EPI_L2_HINT": "1"}, {"MOM_EPI_L2_HINT": "3"},
         {"MOM_EPI_L2_HINT": "3", "MOM_CTA_GROUP": "1"}, {"MOM_EPI_L2_HINT": "1", "MOM_GROUP_M_A": "32"},
         {"MOM_RASTER_B_COLS": "1"}, {"MOM_RASTER_B_COLS": "3"}, {"MOM_RASTER_B_COLS": "8", "MOM_CTA_GROUP": "1"}]
ALL = sorted({k for v in KNOBS for k in v})


def test_knobs_are_bit_neutral(cuda_device):
    S, d, I, C = 1500, 512, 1160, 700
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    x = synth.hidden(S, d, cuda_device, bf)
    res = synth.hidden(S, d, cuda_device, bf, seed=synth.SEED_X + 1)
    old = {k: os.environ.get(k) for k in ALL}
    outs = []
    try:
        for knob in KNOBS:
            for k in ALL:
                os.environ.pop(k, None)
            os.environ.update(knob)
            o = torch.empty_like(x)
            _mom.mlp_minseq_fwd(x, res, wg, wu, wd, o, C)
            torch.cuda.synchronize()
            outs.append(o)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for knob, o in zip(KNOBS, outs):
        assert torch.equal(o, outs[0]), knob


# the non-K-split family (variants 0-3) shares one summation order; the default (5) is tested in
# test_gemv_ksplit_down_variants
GEMV_KNOBS = [{"MOM_GEMV_VARIANT": "2"}, {"MOM_GEMV_VARIANT": "0"}, {"MOM_GEMV_VARIANT": "2", "MOM_GEMV_PDL": "0"},
              {"MOM_GEMV_VARIANT": "2", "MOM_GEMV_PREFETCH": "2"}, {"MOM_GEMV_VARIANT": "0", "MOM_GEMV_PDL": "0"},
              {"MOM_GEMV_VARIANT": "1"}, {"MOM_GEMV_VARIANT": "3"}]
GEMV_ALL = sorted({k for v in GEMV_KNOBS for k in v})


@pytest.mark.parametrize("variant", ["5", "6"])
@pytest.mark.parametrize("d,I", [(4096, 14336), (3584, 18944), (520, 1160), (256, 688)])
def test_gemv_ksplit_down_variants(cuda_device, variant, d, I):
    """MOM_GEMV_VARIANT=5 / 6: the down GEMV K-split over 2 / 4 warps per row group (a different, fixed
    summation order): bit-identical with and without PDL, and within the bf16 bar of the oracle."""
    import oracle
    from tests.parity import TOL_BF16, check_close
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    x = synth.hidden(1, d, cuda_device, bf)[0]
    res = synth.hidden(1, d, cuda_device, bf, seed=synth.SEED_X + 1)[0]
    outs = []
    old = {k: os.environ.get(k) for k in ("MOM_GEMV_VARIANT", "MOM_GEMV_PDL")}
    try:
        for knob in ({"MOM_GEMV_VARIANT": variant}, {"MOM_GEMV_VARIANT": variant, "MOM_GEMV_PDL": "0"}):
            os.environ.pop("MOM_GEMV_PDL", None)
            os.environ.update(knob)
            y = torch.empty_like(x)
            _mom.mlp_last_token(x, res, wg, wu, wd, y)
            torch.cuda.synchronize()
            outs.append(y)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert torch.equal(outs[0], outs[1])
    ref = oracle.mlp_rows(x.cpu()[None], res.cpu()[None], wg.cpu(), wu.cpu(), wd.cpu(), [0])[0]
    check_close(outs[0].cpu(), ref, TOL_BF16, f"last-token K-split{variant} d={d} I={I}")


@pytest.mark.parametrize("d,I", [(4096, 14336), (520, 1160)])
def test_gemv_knobs_are_bit_neutral(cuda_device, d, I):
    """Last-token GEMV shapes (rows per warp step, loads in flight, PDL, L2 prefetch) keep each
    row's summation order: the output is bitwise identical for every setting."""
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    x = synth.hidden(1, d, cuda_device, bf)[0]
    old = {k: os.environ.get(k) for k in GEMV_ALL}
    outs = []
    try:
        for knob in GEMV_KNOBS:
            for k in GEMV_ALL:
                os.environ.pop(k, None)
            os.environ.update(knob)
            y = torch.empty_like(x)
            _mom.mlp_last_token(x, x, wg, wu, wd, y)
            torch.cuda.synchronize()
            outs.append(y)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for knob, y in zip(GEMV_KNOBS, outs):
        assert torch.equal(y, outs[0]), knob


@pytest.mark.parametrize("cg", ["2", "1"])
def test_half_width_tail_tiles(cuda_device, cg):
    """Phase A's last partial wave runs as half-width (64-column) tiles when it fills at most half
    of the clusters (S=2000, C=600, I=4096: 96 tiles on 74 pairs -> 22 tiles become 44 halves; 1-CTA:
    160 on 148 -> 12 -> 24).  Same K order per element: bitwise equal to full tiles, and to the oracle."""
    import oracle
    from tests.parity import TOL_BF16, check_close
    S, d, I, C = 2000, 512, 4096, 600
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    x = synth.hidden(S, d, cuda_device, bf)
    old = {k: os.environ.get(k) for k in ("MOM_HALF_TAIL", "MOM_CTA_GROUP")}
    outs = []
    try:
        os.environ["MOM_CTA_GROUP"] = cg
        for ht in ("1", "0"):
            os.environ["MOM_HALF_TAIL"] = ht
            o = torch.empty_like(x)
            _mom.mlp_minseq_fwd(x, x, wg, wu, wd, o, C)
            torch.cuda.synchronize()
            outs.append(o)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert torch.equal(outs[0], outs[1])
    rows = [0, 599, 600, 1199, 1200, 1799, 1800, 1999] + list(range(3, S, 97))
    xc = x.cpu()
    ref = oracle.mlp_rows(xc, xc, wg.cpu(), wu.cpu(), wd.cpu(), rows)
    check_close(outs[0].cpu()[rows], ref, TOL_BF16, "half-width tail tiles")


@pytest.mark.parametrize("fast", ["1", "0"])
def test_silu_quotient_variants_vs_oracle(cuda_device, fast):
    """MOM_FAST_SILU: the phase-A SiLU quotient by rcp.approx (default) or IEEE division.  Not a
    bit-neutral knob (<= 2 fp32 ulp before the bf16 rounding of H); both meet the oracle bar."""
    import oracle
    from tests.parity import TOL_BF16, check_close
    S, d, I, C = 1500, 512, 1160, 700
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    x = synth.hidden(S, d, cuda_device, bf)
    old = os.environ.get("MOM_FAST_SILU")
    try:
        os.environ["MOM_FAST_SILU"] = fast
        o = torch.empty_like(x)
        _mom.mlp_minseq_fwd(x, x, wg, wu, wd, o, C)
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("MOM_FAST_SILU", None)
        else:
            os.environ["MOM_FAST_SILU"] = old
    rows = [0, 699, 700, 1399, 1400, 1499] + list(range(5, S, 61))
    xc = x.cpu()
    check_close(o.cpu()[rows], oracle.mlp_rows(xc, xc, wg.cpu(), wu.cpu(), wd.cpu(), rows), TOL_BF16,
                f"MOM_FAST_SILU={fast}")
