#!/usr/bin/env python
"""LRU model of phase B's L2 behaviour (a MODEL, not a measurement): which operand's re-reads make
phase B move ~1.3 GB of DRAM for 0.35 GB of operands.  74 clusters run tiles t = c, c+74, ... in
lockstep; a tile streams 224 K-blocks, each reading one 32 KB slice of its H panel (A, row block m) and
one of its W_down panel (B, column block n); its epilogue reads the residual and writes the output
(128 KB each).  L2 = LRU over 32 KB slices (126 MB; no sets, no die split).  Prints DRAM read bytes
per operand for the current raster (group_m row blocks, m fastest) and for alternatives."""
import argparse
from collections import OrderedDict

ap = argparse.ArgumentParser()
ap.add_argument("--C", type=int, default=8192)
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--I", type=int, default=14336)
ap.add_argument("--l2_mb", type=float, default=126.0)
args = ap.parse_args()

SL = 32 * 1024
m_tiles, n_tiles, kb = args.C // 256, args.d // 256, args.I // 64
clusters = 74


def tiles_grouped(G):
    out = []
    for g in range(0, m_tiles, G):
        gm = min(G, m_tiles - g)
        for local in range(gm * n_tiles):
            out.append((g + local % gm, local // gm))
    return out


def run(order, reverse_k=lambda m, n: False, l2_mb=args.l2_mb, keep=None):
    cap = int(l2_mb * 1024 * 1024 / SL)
    lru = OrderedDict()
    miss = {"A": 0, "B": 0, "epi": 0}
    def touch(key, kind):
        if key in lru:
            lru.move_to_end(key)
            return
        miss[kind] += 1
        lru[key] = 1
        while len(lru) > cap:
            lru.popitem(last=False)
    waves = [order[i:i + clusters] for i in range(0, len(order), clusters)]
    for w in waves:
        for k in range(kb):
            for (m, n) in w:
                kk = kb - 1 - k if reverse_k(m, n) else k
                touch(("A", m, kk), "A")
                touch(("B", n, kk), "B")
        for (m, n) in w:  # epilogue: residual read (4 slices), output write (4 slices), streaming
            for q in range(8):
                touch(("E", m, n, q), "epi")
    gb = lambda s: s * SL / 1e9
    return {k: round(gb(v), 3) for k, v in miss.items()}


print(f"operands: H {m_tiles * kb * SL / 1e9:.3f} GB, W_down {n_tiles * kb * SL / 1e9:.3f} GB")
for G in (4, 8, 16, 32):
    print(f"group_m={G:2d} (m fastest)            ", run(tiles_grouped(G)))
for G in (8,):
    print(f"group_m={G:2d} + K reversed on odd n   ", run(tiles_grouped(G), lambda m, n: n % 2 == 1))
    print(f"group_m={G:2d} + K reversed on odd m   ", run(tiles_grouped(G), lambda m, n: m % 2 == 1))


def tiles_col_grouped(GN):
    """groups of GN column blocks (n), n fastest within a group, all m"""
    out = []
    for g in range(0, n_tiles, GN):
        gn = min(GN, n_tiles - g)
        for local in range(gn * m_tiles):
            out.append((local // gn, g + local % gn))
    return out


print("--- alternatives")
for G in (4, 8, 16):
    print(f"group_m={G:2d} K rev odd n             ", run(tiles_grouped(G), lambda m, n: n % 2 == 1))
for GN in (2, 4, 8):
    print(f"col groups of {GN} (n fastest)        ", run(tiles_col_grouped(GN)))
    print(f"col groups of {GN} + K rev odd n      ", run(tiles_col_grouped(GN), lambda m, n: n % 2 == 1))


def run_wave_rev(order, l2_mb=args.l2_mb):
    """K reversed on every other WAVE (not C-invariant: a lower bound for K-direction tricks)."""
    cap = int(l2_mb * 1024 * 1024 / SL)
    lru = OrderedDict()
    miss = {"A": 0, "B": 0, "epi": 0}
    def touch(key, kind):
        if key in lru:
            lru.move_to_end(key); return
        miss[kind] += 1; lru[key] = 1
        while len(lru) > cap: lru.popitem(last=False)
    waves = [order[i:i + clusters] for i in range(0, len(order), clusters)]
    for wi, w in enumerate(waves):
        for k in range(kb):
            kk = kb - 1 - k if wi % 2 else k
            for (m, n) in w:
                touch(("A", m, kk), "A"); touch(("B", n, kk), "B")
        for (m, n) in w:
            for q in range(8): touch(("E", m, n, q), "epi")
    return {k: round(v * SL / 1e9, 3) for k, v in miss.items()}


print("--- lower bounds (wave-parity K reversal, not C-invariant)")
for G in (4, 8, 16):
    print(f"group_m={G:2d} wave-rev                ", run_wave_rev(tiles_grouped(G)))
for GN in (4, 8):
    print(f"col groups of {GN} wave-rev           ", run_wave_rev(tiles_col_grouped(GN)))
