"""f1: the all-gather fused into the phase-B epilogue (mom_mlp_minseq_fwd_gather).

On one GPU: (1) local "peer" buffers receive bit-identical rows and nothing else; (2) two
processes on the same GPU exchange cudaIpcMemHandles of their gathered buffers (over a gloo
group), each runs its token shard with the other's buffer as a peer, and both end with the
full gathered output equal, bitwise, to the unsharded computation.  Only the NVLink transport
is not exercised here (one GPU per gpurun box); the store path and the IPC plumbing are."""
from __future__ import annotations

import os
import socket

import pytest
import torch

import synth
from paper_2504_12526_b200 import _mom

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _env():
    keys = ("MOM_FUSED", "MOM_CTA_GROUP", "MOM_GATHER_FORWARD")
    old = {k: os.environ.get(k) for k in keys}
    yield
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("fused,cg,fwd", [("0", "2", "1"), ("0", "2", "0"), ("1", "2", "1"), ("0", "1", "1")])
def test_gather_into_local_peer_buffers(cuda_device, fused, cg, fwd):
    """fwd=1: rows of mini-sequence i-1 are forwarded by warps 2-3 during mini-sequence i's phase A,
    the last mini-sequence's rows by its phase-B epilogue; fwd=0: every epilogue stores to peers."""
    os.environ["MOM_FUSED"], os.environ["MOM_CTA_GROUP"], os.environ["MOM_GATHER_FORWARD"] = fused, cg, fwd
    S, d, I, C, world, rank = 700, 512, 1024, 256, 4, 2
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    x = synth.hidden(S, d, cuda_device, bf)
    ref = torch.empty_like(x)
    _mom.mlp_minseq_fwd(x, x, wg, wu, wd, ref, C)
    sentinel = torch.full((world * S, d), -7.0, dtype=bf, device=cuda_device)
    mine = sentinel.clone()
    peers = [sentinel.clone() for _ in range(3)]
    sl = slice(rank * S, (rank + 1) * S)
    _mom.mlp_minseq_fwd_gather(x, x, wg, wu, wd, mine[sl], [p[sl] for p in peers], C)
    torch.cuda.synchronize()
    for buf in [mine] + peers:
        assert torch.equal(buf[sl], ref)
        assert torch.equal(buf[:rank * S], sentinel[:rank * S]) and torch.equal(buf[(rank + 1) * S:],
                                                                                  sentinel[(rank + 1) * S:])


@pytest.mark.parametrize("fwd", ["1", "0"])
def test_from_host_gather_into_local_peer_buffers(cuda_device, fwd):
    """The end-to-end entry of token-sharded runs: input streamed from pinned host memory per
    mini-sequence (x_free prefetch event), output rows stored to every peer buffer too."""
    os.environ["MOM_GATHER_FORWARD"] = fwd
    S, d, I, C, world, rank = 700, 512, 1024, 256, 3, 1
    bf = torch.bfloat16
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, bf)
    x = synth.hidden(S, d, cuda_device, bf)
    ref = torch.empty_like(x)
    _mom.mlp_minseq_fwd(x, x, wg, wu, wd, ref, C)
    sentinel = torch.full((world * S, d), -3.0, dtype=bf, device=cuda_device)
    mine = sentinel.clone()
    peers = [sentinel.clone() for _ in range(world - 1)]
    sl = slice(rank * S, (rank + 1) * S)
    x_host = x.cpu().pin_memory()
    x_dev = torch.zeros_like(x)
    free = torch.cuda.Event()
    compute, cp = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(compute):
        free.record(compute)
        _mom.mlp_minseq_fwd_from_host_gather(x_host, x_dev, x_dev, wg, wu, wd, mine[sl], [p[sl] for p in peers], C,
                                             stream=compute, copy_stream=cp, x_free=free)
    torch.cuda.synchronize()
    assert torch.equal(x_dev, x)
    for buf in [mine] + peers:
        assert torch.equal(buf[sl], ref)
        assert torch.equal(buf[:rank * S], sentinel[:rank * S]) and torch.equal(buf[(rank + 1) * S:],
                                                                                  sentinel[(rank + 1) * S:])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, S, d, I, C, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        bf = torch.bfloat16
        wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
        xs = [synth.hidden(S, d, dev, bf, seed=synth.SEED_X + r) for r in range(world)]
        refs = []
        for r in range(world):  # the unsharded result, computed locally with the plain path
            o = torch.empty_like(xs[r])
            _mom.mlp_minseq_fwd(xs[r], xs[r], wg, wu, wd, o, C)
            refs.append(o)
        gathered = torch.zeros((world * S, d), dtype=bf, device=dev)
        torch.cuda.synchronize()
        handle = _mom.ipc_get_handle(gathered)
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        peers = {}
        for r in range(world):
            if r != rank:
                peers[r] = _mom.ipc_open_handle(*handles[r])
        sl = slice(rank * S, (rank + 1) * S)
        row_bytes = d * 2
        peer_ptrs = [peers[r] + rank * S * row_bytes for r in sorted(peers)]
        _mom.mlp_minseq_fwd_gather(xs[rank], xs[rank], wg, wu, wd, gathered[sl], peer_ptrs, C)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's peer stores are complete
        ok = torch.equal(gathered, torch.cat(refs))
        dist.barrier()
        for r, ptr in peers.items():
            _mom.ipc_close(ptr, handles[r][1])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gather_two_processes_ipc(cuda_device):
    import torch.multiprocessing as mp
    world, S, d, I, C = 2, 600, 256, 512, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, S, d, I, C, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == [(0, True), (1, True)]
