"""Host-side orchestration of Alg. 1 over a stack of L layers, for BASELINE configs 3-5.

Pure control flow around the C-ABI calls (no arithmetic of the method runs here): per layer l
  1. attention is out of scope: a caller-supplied stand-in writes the layer's K/V into
     slot l % 2 of a two-slot device ring (the slot is reused only after its previous offload
     finished -- event-gated, so the caching allocator never recycles memory under a live copy);
  2. mom_kv_offload copies it to the pinned host mirror of layer l on the copy stream,
     overlapping the MLP;
  3. non-final layers: mom_mlp_minseq_fwd in place, x <- x + MLP(x), and, when the
     tokens are sharded over N GPUs, mom_allgather_rows rebuilds the [N*S, d] rows;
  4. final layer: mom_mlp_last_token on the last token, mom_lm_head_last;
  5. after the head, mom_kv_reload brings every layer's K/V back to the device, one
     event per layer (f4: a decode step may start layer l as soon as its K/V is back).
Token sharding: rank r owns rows [r*S_r, (r+1)*S_r) of N*S_r (padded) rows.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from . import _mom


def shard_rows(S_total: int, world: int, rank: int):
    """Contiguous token shard of `rank`: (start, count, padded_total).  S_total is padded up to
    world * ceil(S_total / world) rows; pad rows are computed and dropped (rows are independent)."""
    if world < 1 or not 0 <= rank < world or S_total < 1:
        raise ValueError("bad shard arguments")
    per = math.ceil(S_total / world)
    return rank * per, per, per * world


def last_token_owner(S_total: int, world: int) -> int:
    """Rank holding token S_total - 1 (runs the final-layer GEMVs and the head)."""
    per = math.ceil(S_total / world)
    return (S_total - 1) // per


@dataclass
class StackResult:
    y_last: torch.Tensor | None
    logits: torch.Tensor | None
    argmax: torch.Tensor | None
    kv_host: list = field(default_factory=list)
    kv_dev: list = field(default_factory=list)
    launches: int = 0
    # f4: one event per layer, recorded on the copy stream when that layer's K/V is back on the
    # device; a decode step can start layer l after reload_done[l] while layers > l still stream
    reload_done: list = field(default_factory=list)


class PrefillStack:
    """MOM prefill of the MLP path over L layers on one GPU (or one token shard of N)."""

    def __init__(self, weights, w_head, norm_gain, eps, S_local, minseq_len, kv_shape, device,
                 world=1, rank=0, comm=None, S_total=None, offload=True, reload=True, peers=None,
                 pipelined_reload=False):
        self.weights = weights            # list of (w_gate, w_up, w_down), layer 0..L-1
        self.L = len(weights)
        self.wh, self.gain, self.eps = w_head, norm_gain, eps
        self.S, self.C = S_local, minseq_len
        self.world, self.rank, self.comm = world, rank, comm
        # f1: peers' x buffers (NVLink-mapped, offset to this rank's shard rows); the phase-B
        # epilogue stores every output row there, so no separate all-gather runs
        self.peers = list(peers or [])
        self.barrier_scratch = torch.zeros(1, dtype=torch.int32, device=device) if world > 1 else None
        self.S_total = S_total if S_total is not None else S_local * world
        self.device = device
        wg0 = weights[0][0]
        self.dtype = wg0.dtype
        self.I, self.d = wg0.shape
        self.V = w_head.shape[0]
        self.ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S_local, self.d, self.I, minseq_len, self.dtype),
                              dtype=torch.uint8, device=device)
        self.ws_last = torch.empty(_mom.lib().mom_mlp_last_token_workspace_bytes(self.I), dtype=torch.uint8,
                                   device=device)
        self.ws_head = torch.empty(_mom.lib().mom_lm_head_workspace_bytes(self.V), dtype=torch.uint8, device=device)
        self.offload, self.reload = offload, reload and offload
        # f4: when True, run() does not join the copy stream after the reload; the caller waits
        # on StackResult.reload_done[l] per layer (decode of layer l overlaps the H2D of l+1..)
        self.pipelined_reload = pipelined_reload
        self.kv_shape = kv_shape
        self.kv_ring = [torch.empty(kv_shape, dtype=self.dtype, device=device) for _ in range(2)] if offload else []
        self.kv_host = [torch.empty(kv_shape, dtype=self.dtype, pin_memory=True) for _ in range(self.L)] if offload else []
        self.kv_dev = [torch.empty(kv_shape, dtype=self.dtype, device=device) for _ in range(self.L)] if self.reload else []
        self.y = torch.empty(self.d, dtype=self.dtype, device=device)
        self.logits = torch.empty(self.V, dtype=torch.float32, device=device)
        self.argmax = torch.empty(1, dtype=torch.int32, device=device)
        self.owner = last_token_owner(self.S_total, world)

    def run(self, x, kv_fill=None, compute=None, copy=None, on_layer=None):
        """x: [world * S_local, d] device tensor (this rank's shard at rows rank*S_local), updated in
        place to the final layer's input.  kv_fill(l, slot) writes layer l's stand-in K/V on the
        current stream.  on_layer(l, x) is called (host side, after enqueueing) before layer l's MLP
        -- tests use it to snapshot teacher-forcing inputs.  Returns a StackResult."""
        compute = compute or torch.cuda.current_stream(self.device)
        copy = copy or torch.cuda.Stream(self.device)
        ev_off = [torch.cuda.Event() for _ in range(self.L)]
        shard = x[self.rank * self.S:(self.rank + 1) * self.S]
        launches = 0
        with torch.cuda.stream(compute):
            for l in range(self.L):
                if self.offload:
                    slot = self.kv_ring[l % 2]
                    if l >= 2:
                        compute.wait_event(ev_off[l - 2])   # slot reuse only after its D2H finished
                    if kv_fill is not None:
                        kv_fill(l, slot)
                    _mom.kv_offload(slot, self.kv_host[l], compute, copy, ev_off[l])          # a9
                if on_layer is not None:
                    on_layer(l, x)
                wg, wu, wd = self.weights[l]
                if l < self.L - 1:
                    if self.world > 1 and self.peers:  # a1-a5 + a11 fused (f1)
                        _mom.mlp_minseq_fwd_gather(shard, shard, wg, wu, wd, shard, self.peers, self.C, self.ws,
                                                   compute)
                        _mom.nccl_barrier(self.comm, self.barrier_scratch, compute)
                    else:
                        _mom.mlp_minseq_fwd(shard, shard, wg, wu, wd, shard, self.C, self.ws, compute)  # a1-a5
                        if self.world > 1:
                            _mom.allgather_rows(x, self.S, self.comm, self.rank, self.world, compute)  # a11
                    launches += 2 * math.ceil(self.S / self.C)
                elif self.rank == self.owner:
                    last = x[self.S_total - 1]
                    _mom.mlp_last_token(last, last, wg, wu, wd, self.y, self.ws_last, compute)     # a6
                    _mom.lm_head_last(self.y, self.gain, self.eps, self.wh, self.logits, self.argmax,
                                      self.ws_head, compute)                                       # a7-a8
                    launches += 4
            reload_done = []
            if self.reload:
                copy.wait_stream(compute)  # Alg. 1: after the head
                for l in range(self.L):     # layer order = decode order (f4: per-layer completion)
                    ev = torch.cuda.Event()
                    _mom.kv_reload(self.kv_host[l], self.kv_dev[l], copy, ev)                      # a10
                    reload_done.append(ev)
                if not self.pipelined_reload:
                    compute.wait_stream(copy)
        own = self.rank == self.owner
        return StackResult(self.y if own else None, self.logits if own else None, self.argmax if own else None,
                           self.kv_host, self.kv_dev, launches, reload_done)
