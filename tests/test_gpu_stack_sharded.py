"""Token-sharded layer stack (BASELINE config 5's split) at world size 2, as two
(and 4) processes on the one GPU of a gpurun box: real cudaIpc handles for both gathered buffers, the f1
peer stores of the phase-B epilogue, a gloo host barrier per layer (comm=None test mode of
PrefillStack).  Mini-sequences are independent, so every gathered row, the
last-token MLP output, the logits and the argmax must equal the one-GPU stack's BITWISE (the GPU-only
exact invariant of SURVEY §8(c)); the one-GPU stack is itself oracle-checked in test_gpu_stack.py.
Also covered: a padded (non-divisible) S_total, the ping-pong buffer order, per-rank KV offload
bytes, and two consecutive runs (the second reuses ring, host mirrors and peer mappings)."""
from __future__ import annotations

import os
import socket

import pytest
import torch

import synth
from paper_2504_12526_b200.stack import PrefillStack, last_token_owner, shard_rows

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model(d, I, V, L, dev):
    bf = torch.bfloat16
    return ([synth.mlp_weights(d, I, l, dev, bf) for l in range(L)], synth.head_weight(V, d, dev, bf),
            synth.norm_gain(d, dev, bf))


def _kv_fill_for(base, row0):
    def fill(l, slot):  # stand-in K/V of this rank's rows: global row ids stamped into column 1
        slot.copy_(base)
        v = slot.view(torch.int16)
        v[:, 0] = l
        v[:, 1] = (torch.arange(slot.shape[0], device=slot.device, dtype=torch.int32) + row0).to(torch.int16)
    return fill


def _worker(rank, world, port, cfg, q, early="off"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, I, V, L, S_total, C, d_kv, eps = cfg
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        bf = torch.bfloat16
        weights, wh, gain = _model(d, I, V, L, dev)
        x_full = synth.hidden(S_total, d, dev, bf)
        # one-GPU reference stack on all S_total rows (computed by every rank, locally)
        ref_stack = PrefillStack(weights, wh, gain, eps, S_total, C, (S_total, 2 * d_kv), dev, offload=False)
        x_ref = x_full.clone()
        ref = ref_stack.run(x_ref)
        torch.cuda.synchronize()
        # the token-sharded stack
        start, per, padded = shard_rows(S_total, world, rank)
        x_mine = torch.zeros((per, d), dtype=bf, device=dev)
        n_real = max(0, min(per, S_total - start))
        x_mine[:n_real] = x_full[start:start + n_real]
        base = synth.kv_standin(per, d_kv, 0, dev, bf)
        st = PrefillStack(weights, wh, gain, eps, per, C, (per, 2 * d_kv), dev, world=world, rank=rank,
                          comm=None, S_total=S_total, gather="fused", early_reload=early)
        seen = []
        ok = True
        for rep in range(2):
            for b in st.xbuf:
                b.fill_(-5.0)  # sentinel: every row must be rewritten by its owner's stores
            res = st.run(x_mine, _kv_fill_for(base, start), on_layer=lambda l, buf: seen.append(buf.data_ptr()))
            torch.cuda.synchronize()
            dist.barrier()
            if L > 1:
                ok &= torch.equal(res.x_final[:S_total], x_ref)
            assert seen[:L] == [st.xbuf[l % 2].data_ptr() for l in range(L)]
            seen.clear()
            owner = last_token_owner(S_total, world)
            if rank == owner:
                ok &= torch.equal(res.y_last, ref.y_last) and torch.equal(res.logits, ref.logits)
                ok &= int(res.argmax.item()) == int(ref.argmax.item())
            else:
                ok &= res.y_last is None
            for l in range(L):
                h = res.kv_host[l].view(torch.int16)
                ok &= bool((h[:, 0] == l).all())
                ok &= torch.equal(h[:, 1].to(torch.int32), torch.arange(per, dtype=torch.int32) + start)
                ok &= torch.equal(res.kv_dev[l], res.kv_host[l].to(dev))
        dist.barrier()
        st.close()
        q.put((rank, bool(ok)))
    except Exception as e:  # report instead of hanging the peer
        q.put((rank, f"error: {e!r}"))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,S_total,early", [(2, 1536, "off"), (2, 1501, "off"), (4, 2050, "off"),
                                                 (2, 1536, 1 << 40)])
def test_sharded_stack_equals_one_gpu_bitwise(cuda_device, world, S_total, early):
    """world 4: every rank stores each output row to 3 peers (and forwards the previous mini-sequence's
    rows to 3 peers); S_total = 2050 pads the last shard by 2 rows; the last case reloads every layer's
    K/V right after its offload (f4, unlimited budget) on every rank."""
    import torch.multiprocessing as mp
    cfg = (256, 512, 1000, 4, S_total, 256, 64, 1e-5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q, early)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    assert res == [(r, True) for r in range(world)], res
    for p in procs:
        assert p.exitcode == 0
