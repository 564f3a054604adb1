"""CPU tests of bench.py's host-side arithmetic: the phase-B tile-width model it mirrors from the library
(wave quantisation on 74 CTA pairs), and the in-kernel-trace parser that turns %globaltimer / clock64
stamps into an SM clock, MMA-issue efficiency and FLOP per SM-cycle."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


@pytest.mark.parametrize("d,S,expect", [(4096, 8192, 256), (3584, 8192, 224), (5120, 8192, 256), (5120, 7544, 160),
                                        (256, 1024, 128)])
def test_phase_b_width_model(d, S, expect):
    m_tiles = -(-S // 256)
    nb = bench.phase_b_width(m_tiles, d, 74)
    assert nb == expect and nb % 32 == 0 and (d % nb == 0 or nb == 256)
    waves = lambda w: -(-(m_tiles * -(-d // w)) // 74) * w  # noqa: E731 -- the model's cost
    assert waves(nb) <= waves(256)


def test_trace_efficiency_on_synthetic_stamps():
    """One call of one mini-sequence (S = C = 8192, d 4096, I 14336): phase A and B launches whose CTAs
    all issue MMAs back to back at 1.0 GHz for exactly the ideal number of cycles -> efficiency 1.0,
    clock 1000 MHz, and FLOP/SM/cycle = the algorithmic FLOP over (SMs x cycles incl. the tail)."""
    S = C = 8192
    d, I, sms = 4096, 14336, 148
    t = np.zeros((2, 160, 8), dtype=np.int64)
    kbA, kbB = d // 64, I // 64
    m_tiles, nA = S // 256, I // 128
    T = m_tiles * nA
    R = T % 74
    idealA = (T - R) // 74 * kbA * 512 + kbA * 256 if 0 < 2 * R <= 74 else -(-T // 74) * kbA * 512
    idealB = -(-(m_tiles * (d // 256)) // 74) * kbB * 512
    t0 = 1_000_000
    for j, ideal in ((0, idealA), (1, idealB)):
        start = t0 if j == 0 else t0 + idealA + 5_000  # 5 us gap A -> B (ns = cycles at 1 GHz)
        for c in range(sms):
            t[j, c, 0] = start - 100
            t[j, c, 1] = start            # first MMA (ns)
            t[j, c, 2] = start + ideal    # last MMA (ns)
            t[j, c, 3] = start + ideal + 1_000  # exit
            t[j, c, 4] = 10_000
            t[j, c, 5] = 10_000 + ideal   # clock64 cycles over the MMA span: 1 GHz
    r = bench.trace_efficiency(t, S, C, d, I, sms)
    assert r["phaseA_mhz"] == 1000 and r["phaseB_mhz"] == 1000
    assert r["phaseA_mma_issue_efficiency"] == pytest.approx(1.0, abs=1e-4)
    assert r["phaseB_mma_issue_efficiency"] == pytest.approx(1.0, abs=1e-4)
    assert r["A_to_B_gap_us"] == pytest.approx(5.0, abs=1e-6)
    fpc_a = 4.0 * S * d * I / (sms * (idealA + 1_000))
    assert r["phaseA_flop_per_sm_cycle"] == pytest.approx(fpc_a, rel=1e-3)
    assert r["mlp_step_mma_issue_efficiency"] == pytest.approx((idealA + idealB) / (idealA + 5_000 + idealB), abs=1e-4)


def test_default_steps_make_a_sustained_region(monkeypatch):
    """No flags: 200 timed config-2 steps (~17 ms each -> >= 3 s, the region length from which bench.py
    divides by the sustained peak); --stack: 20; an explicit --steps wins."""
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    assert bench.resolve_defaults(bench.parse_args()).steps == 200
    assert 200 * 16.4e-3 >= 3.0
    monkeypatch.setattr(sys, "argv", ["bench.py", "--stack"])
    assert bench.resolve_defaults(bench.parse_args()).steps == 20
    monkeypatch.setattr(sys, "argv", ["bench.py", "--steps", "7"])
    assert bench.resolve_defaults(bench.parse_args()).steps == 7
