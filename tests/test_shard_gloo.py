"""World-size-2 CPU (gloo) test of the token-sharded multi-GPU host logic:
shard plan, last-token owner, and gather order.  Each rank computes its shard's rows with the
ORACLE (the CUDA path needs GPUs and NCCL; its in-place all-gather is exercised on the GPU), the
rows are all-gathered in rank order, and the result must equal the unsharded computation
bitwise (rows are independent) -- including a padded (non-divisible) S."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2504_12526_b200.stack import last_token_owner, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(S, d, I):
    r = np.random.default_rng(5)
    x = r.standard_normal((S, d)).astype(np.float32)
    wg = (r.standard_normal((I, d)) * 0.2).astype(np.float32)
    wu = (r.standard_normal((I, d)) * 0.2).astype(np.float32)
    wd = (r.standard_normal((d, I)) * 0.2).astype(np.float32)
    return x, wg, wu, wd


def _worker(rank, world, port, S, d, I, C, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, wg, wu, wd = _inputs(S, d, I)
        start, per, padded = shard_rows(S, world, rank)
        xp = np.zeros((padded, d), np.float32)
        xp[:S] = x
        mine = oracle.mlp_minseq(xp[start:start + per], xp[start:start + per], wg, wu, wd, C=C, nthreads=1)
        parts = [torch.empty((per, d), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        gathered = torch.cat(parts).numpy()[:S]
        owner = last_token_owner(S, world)
        q.put((rank, gathered.tobytes(), owner, start, per, padded))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S", [64, 67])
def test_token_shard_gather_equals_unsharded(S):
    world, d, I, C = 2, 16, 24, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, d, I, C, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, wg, wu, wd = _inputs(S, d, I)
    ref = oracle.mlp_minseq(x, x, wg, wu, wd, C=S)
    res.sort()
    for rank, blob, owner, start, per, padded in res:
        assert blob == ref.tobytes(), rank
        assert owner == (S - 1) // per and start == rank * per and padded == per * world


def test_shard_plan_edges():
    assert shard_rows(455000, 8, 7) == (7 * 56875, 56875, 455000)
    assert shard_rows(10, 4, 3) == (9, 3, 12)
    assert last_token_owner(455000, 8) == 7
    assert last_token_owner(10, 4) == 3
    assert last_token_owner(9, 4) == 2  # per = 3: rows 6..8 on rank 2, rank 3 holds only padding
    with pytest.raises(ValueError):
        shard_rows(10, 0, 0)


# ---------------------------------------------------------------- f2: vocab-sharded LM head protocol
def _pack_key(v: np.float32, idx: int) -> int:
    """The kernels' argmax key (gemv.cu pack_key, include/mom.h f2): order-preserving float -> u32 in
    the high word, complemented GLOBAL vocab index in the low word, so the u64 max is the largest
    logit and, among equal logits, the lowest index."""
    b = int(np.float32(v).view(np.uint32))
    b = (~b & 0xFFFFFFFF) if (b & 0x80000000) else (b | 0x80000000)
    return (b << 32) | (0xFFFFFFFF - idx)


def _head_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V, d = 1000, 32
        r = np.random.default_rng(9)
        h = r.standard_normal(d).astype(np.float32)
        w = (r.standard_normal((V, d)) * 0.1).astype(np.float32)
        w[700] = w[10] = w[int(np.argmax(w @ h))] * 1.0 + 0.5 * h / np.linalg.norm(h)  # a tie across shards
        per = V // world
        lo = rank * per
        logits = oracle.lm_head(h.astype(np.float64), w[lo:lo + per])[0].astype(np.float32)  # fp32 like the kernel
        best = max(_pack_key(v, lo + i) for i, v in enumerate(logits))
        # gloo has no uint64 max: flip the top bit so signed int64 order equals u64 order
        t = torch.tensor([best ^ (1 << 63)], dtype=torch.uint64).view(torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        key = int(t.view(torch.uint64).item()) ^ (1 << 63)
        q.put((rank, 0xFFFFFFFF - (key & 0xFFFFFFFF)))
    finally:
        dist.destroy_process_group()


def test_vocab_sharded_argmax_protocol():
    """f2: each rank reduces its vocab shard to one packed key, one u64 max across the
    ranks gives the global argmax -- ties across shards resolve to the lowest index."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_head_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert {idx for _, idx in res} == {10}  # rows 10 (rank 0) and 700 (rank 1) tie at the max


def test_pack_key_orders_like_floats():
    vals = np.array([-np.inf, -3.5, -1e-30, -0.0, 0.0, 1e-30, 2.0, 2.0, np.inf], np.float32)
    keys = [_pack_key(v, i) for i, v in enumerate(vals)]
    assert keys[7] < keys[6]                     # equal values: the lower index has the larger key
    order = sorted(range(len(vals)), key=lambda i: keys[i])
    assert [float(vals[i]) for i in order] == sorted(float(v) for v in vals)
