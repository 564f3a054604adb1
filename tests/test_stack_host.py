"""Host-side logic of the layer stack and the bench's collective setup, CPU only: the f4 reload budget
(all K/V minus the prefill transient keeps the device at or below Alg. 1's end state), the
token-shard plan of config 5 (56 / 28 / 14 / 7 mini-sequences per rank at N =
1 / 2 / 4 / 8, tails 4440 / 6316 / 7254 / 7723), the ping-pong buffer order, and bench.try_collective at
world size 2 over gloo (a failure on one rank reaches every rank, so all take the same fallback)."""
from __future__ import annotations

import math
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_12526_b200.stack import (early_reload_budget, early_reload_plan, gathered_buffer_index,
                                         last_token_owner, shard_rows)


def test_early_reload_budget_keeps_peak_at_alg1_end_state():
    L, kv, transient = 32, 1_863_680_000, 7_689_601_536   # config 5, N = 1 (bench --stack numbers)
    b = early_reload_budget("auto", L, kv, transient)
    assert b == L * kv - transient
    n = early_reload_plan(L, kv, b)
    assert n == 27 and n * kv <= b < (n + 1) * kv
    # peak during prefill = transient + early-reloaded K/V <= every layer's K/V (Alg. 1's end state)
    assert transient + n * kv <= L * kv
    assert early_reload_budget("off", L, kv, transient) == 0
    assert early_reload_budget("auto", 2, kv, transient) == 0          # K/V smaller than the transient
    assert early_reload_plan(L, kv, 10 ** 15) == L                     # unlimited: every layer early
    # the final layer: x (but its last row) and the MLP workspace are dead, two more layers fit
    x_ws = 455000 * 4096 * 2 + 8192 * 14336 * 2
    assert early_reload_plan(L - 1, kv, b + x_ws) == 29 and transient - x_ws + 29 * kv <= L * kv
    assert early_reload_budget(5 * kv, L, kv, transient) == 5 * kv
    with pytest.raises(ValueError):
        early_reload_budget(-1, L, kv, transient)


@pytest.mark.parametrize("N,M,tail", [(1, 56, 4440), (2, 28, 6316), (4, 14, 7254), (8, 7, 7723)])
def test_config5_shard_plan(N, M, tail):
    S, C = 455000, 8192
    starts = []
    for r in range(N):
        start, per, padded = shard_rows(S, N, r)
        starts.append(start)
        assert per * N == padded >= S and per == S // N           # 455000 divides by 2, 4, 8
        assert math.ceil(per / C) == M and per - (M - 1) * C == tail
    assert starts == [r * (S // N) for r in range(N)]
    assert last_token_owner(S, N) == N - 1


def test_ping_pong_order():
    # layer l reads buffer l % 2 and writes (l + 1) % 2: consecutive layers never write what they read
    for l in range(40):
        assert gathered_buffer_index(l) != gathered_buffer_index(l + 1)
        assert gathered_buffer_index(l + 2) == gathered_buffer_index(l)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = bench.try_collective(lambda: None, world, None)

        def fail_on_1():
            if rank == 1:
                raise RuntimeError("cudaIpcGetMemHandle failed (simulated)")
        why = bench.try_collective(fail_on_1, world, None)
        q.put((rank, ok, why))
    finally:
        dist.destroy_process_group()


def test_try_collective_fallback_reaches_every_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, why in res:
        assert ok is None
        assert why is not None and "simulated" in why, (rank, why)
