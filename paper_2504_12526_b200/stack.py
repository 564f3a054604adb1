"""Host-side orchestration of Alg. 1 over a stack of L layers, for BASELINE configs 3-5.

Pure control flow around the C-ABI calls (no arithmetic of the method runs here): per layer l
  1. attention is out of scope: a caller-supplied stand-in writes the layer's K/V into
     slot l % 2 of a two-slot device ring (the slot is reused only after its previous offload
     finished -- event-gated, so the caching allocator never recycles memory under a live copy);
  2. mom_kv_offload copies it to the pinned host mirror of layer l on the copy stream,
     overlapping the MLP;
  3. non-final layers: mom_mlp_minseq_fwd, x <- x + MLP(x).  One GPU: in place.
     Token-sharded over N GPUs: every rank holds the [N*S_r, d] rows in
     TWO gathered buffers used alternately -- layer l reads buffer l % 2 and writes its output rows
     into buffer (l+1) % 2 of every rank (f1: the phase-B epilogue stores them to the IPC-mapped
     peer buffers; or mom_allgather_rows, the NCCL baseline), then one barrier per layer
     (mom_nccl_barrier, or a host barrier in the one-GPU test mode).  Because no rank starts
     layer l+1 before every rank finished layer l, nothing a rank may still read in buffer l % 2
     (its MLP input; a full model's attention over all rows) is overwritten while it is read;
  4. final layer: mom_mlp_last_token on the last token, mom_lm_head_last on
     the rank that owns token S_total - 1;
  5. after the head, mom_kv_reload brings every layer's K/V back to the device, one
     event per layer (f4: a decode step may start layer l as soon as its K/V is back).
     early_reload (f4, off by default = Alg. 1's order): the H2D of layer j may start as soon as its
     D2H finished, on its own stream (PCIe is full duplex, so it runs beside the next layers'
     offloads and MLPs), for as many layers as a device budget allows.  "auto" budget = all layers'
     K/V minus the prefill transient (x, workspace, K/V ring): the device then never holds more than
     at the end of Alg. 1 (weights + every layer's K/V), the paper's peak, while most of the
     reload leaves the time to first token.  The rest is reloaded after the head, as in Alg. 1.
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


def early_reload_budget(mode, layers: int, kv_bytes: int, transient_bytes: int) -> int:
    """f4: bytes of K/V that may be reloaded before the head.  "off" -> 0 (Alg. 1's order); "auto" ->
    all layers' K/V minus the prefill transient, so the device never holds more than at the end of
    Alg. 1 (weights + every layer's K/V); an int -> that many bytes."""
    if mode == "off":
        return 0
    if mode == "auto":
        return max(0, layers * kv_bytes - transient_bytes)
    b = int(mode)
    if b < 0:
        raise ValueError("early_reload budget must be >= 0")
    return b


def early_reload_plan(layers: int, kv_bytes: int, budget: int) -> int:
    """Number of layers whose reload starts before the head: the first ones, in layer order, while the
    reloaded bytes fit the budget (each right after its own offload)."""
    if kv_bytes <= 0:
        return 0
    return min(layers, budget // kv_bytes)


def gathered_buffer_index(layer: int) -> int:
    """Token-sharded stacks: layer l reads gathered buffer l % 2 and writes buffer (l+1) % 2."""
    return layer % 2


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
    # the final layer's input rows (all N*S_r rows when token-sharded; x itself on one GPU)
    x_final: torch.Tensor | None = None
    copy_stream: torch.cuda.Stream | None = None
    early_reload_bytes: int = 0  # f4: bytes whose reload was enqueued before the head (within the budget)


class PrefillStack:
    """MOM prefill of the MLP path over L layers on one GPU (or one token shard of N).

    Token-sharded (world > 1): `gather` = "fused" maps every peer's two gathered buffers through
    cudaIpc handles exchanged over `group` (torch.distributed) and stores the output rows there from
    the MLP kernels; "nccl" runs mom_allgather_rows after each layer (needs one GPU per rank).
    The per-layer barrier is mom_nccl_barrier on `comm`, or, when comm is None (the one-GPU test
    mode with several ranks on one device), a host barrier over `group`."""

    def __init__(self, weights, w_head, norm_gain, eps, S_local, minseq_len, kv_shape, device,
                 world=1, rank=0, comm=None, S_total=None, offload=True, reload=True, gather="fused",
                 group=None, pipelined_reload=False, early_reload="off", defer_last_offload=True,
                 norm_gains=None, norm_eps=1e-5):
        self.weights = weights            # list of (w_gate, w_up, w_down), layer 0..L-1
        self.L = len(weights)
        self.wh, self.gain, self.eps = w_head, norm_gain, eps
        self.S, self.C = S_local, minseq_len
        self.world, self.rank, self.comm, self.group = world, rank, comm, group
        if gather not in ("fused", "nccl"):
            raise ValueError("gather must be 'fused' or 'nccl'")
        if world > 1 and gather == "nccl" and comm is None:
            raise ValueError("gather='nccl' needs an NCCL communicator")
        self.gather = gather
        # f3 in the stack: the Llama pre-norm block x + MLP(RMSNorm(x) * g_l) per layer, the gains
        # folded into W_gate / W_up once here (2 x I x d extra bytes per layer)
        if norm_gains is not None and world > 1 and gather == "fused":
            raise ValueError("norm_gains with the fused gather is not supported (use gather='nccl')")
        self.norm_eps = norm_eps
        self.S_total = S_total if S_total is not None else S_local * world
        if world > 1 and not (world - 1) * S_local < self.S_total <= world * S_local:
            raise ValueError("S_total must satisfy (world-1)*S_local < S_total <= world*S_local")
        self.device = device
        wg0 = weights[0][0]
        self.dtype = wg0.dtype
        self.I, self.d = wg0.shape
        self.V = w_head.shape[0]
        self.folded = None
        if norm_gains is not None:
            if len(norm_gains) != self.L:
                raise ValueError("one norm gain per layer")
            self.folded = [(_mom.fold_norm_gain(wg, g), _mom.fold_norm_gain(wu, g))
                           for (wg, wu, _), g in zip(weights, norm_gains)]
            ws_bytes = _mom.lib().mom_mlp_minseq_rmsnorm_workspace_bytes(S_local, self.d, self.I, minseq_len,
                                                                         _mom._dt(wg0))
        else:
            ws_bytes = _mom.mlp_minseq_workspace_bytes(S_local, self.d, self.I, minseq_len, self.dtype)
        self.ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
        self.ws_last = torch.empty(_mom.lib().mom_mlp_last_token_workspace_bytes(self.I), dtype=torch.uint8,
                                   device=device)
        self.ws_head = torch.empty(_mom.lib().mom_lm_head_workspace_bytes(self.V), dtype=torch.uint8, device=device)
        self.offload, self.reload = offload, reload and offload
        # f4: when True, run() does not join the copy stream after the reload; the caller waits
        # on StackResult.reload_done[l] per layer (decode of layer l overlaps the H2D of l+1..)
        self.pipelined_reload = pipelined_reload
        self.defer_last_offload = defer_last_offload
        self.kv_shape = kv_shape
        self.kv_ring = [torch.empty(kv_shape, dtype=self.dtype, device=device) for _ in range(2)] if offload else []
        self.kv_host = [torch.empty(kv_shape, dtype=self.dtype, pin_memory=True) for _ in range(self.L)] if offload else []
        self.kv_dev = [torch.empty(kv_shape, dtype=self.dtype, device=device) for _ in range(self.L)] if self.reload else []
        self.y = torch.empty(self.d, dtype=self.dtype, device=device)
        self.logits = torch.empty(self.V, dtype=torch.float32, device=device)
        self.argmax = torch.empty(1, dtype=torch.int32, device=device)
        self.owner = last_token_owner(self.S_total, world)
        self.kv_bytes = math.prod(kv_shape) * torch.empty((), dtype=self.dtype).element_size()
        # device bytes prefill needs beyond the weights that are not part of Alg. 1's end state
        x_bytes = (2 * world if world > 1 else 1) * S_local * self.d * torch.empty((), dtype=self.dtype).element_size()
        self.transient_bytes = self.ws.numel() + len(self.kv_ring) * self.kv_bytes + x_bytes
        self.early_budget = (early_reload_budget(early_reload, self.L, self.kv_bytes, self.transient_bytes)
                             if self.reload else 0)
        # once the last mini-sequence layer is done, only the last row of x is live and the MLP workspace
        # is dead: an "auto" budget grows by their bytes for the final layer (Alg. 1)
        self.final_layer_release = (x_bytes + self.ws.numel()) if (early_reload == "auto" and self.reload) else 0
        self.h2d = torch.cuda.Stream(device) if self.reload else None
        # the previous run's copies (offload into kv_host, reload out of it) must finish before a new
        # run refills the ring and the host mirrors (pipelined_reload leaves them in flight)
        self._prev_copies_done = None
        self.xbuf, self.peers, self._peer_maps = [], [[], []], []
        if world > 1:
            self.barrier_scratch = torch.zeros(1, dtype=torch.int32, device=device)
            self.xbuf = [torch.zeros((world * S_local, self.d), dtype=self.dtype, device=device) for _ in range(2)]
            if gather == "fused":
                self._map_peers()

    # ---------------------------------------------------------------- token-sharded plumbing
    def _map_peers(self):
        """Exchange the cudaIpc handles of both gathered buffers and map every peer's, offset to this
        rank's shard rows (where this rank's phase-B epilogue stores its output rows)."""
        import torch.distributed as dist
        try:
            mine = [_mom.ipc_get_handle(b) for b in self.xbuf]
            err = None
        except _mom.MomError as e:  # every rank must still reach the all_gather below
            mine, err = None, e
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=self.group)
        if err is not None:
            raise err
        if any(h is None for h in handles):
            raise RuntimeError("a peer could not export its gathered buffers (cudaIpcGetMemHandle)")
        shard_off = self.rank * self.S * self.d * self.xbuf[0].element_size()
        for b in range(2):
            for r in range(self.world):
                if r == self.rank:
                    continue
                h, off = handles[r][b]
                ptr = _mom.ipc_open_handle(h, off)
                self._peer_maps.append((ptr, off))
                self.peers[b].append(ptr + shard_off)

    def close(self, barrier: bool = True):
        """Unmap the peers' buffers (collective: every rank calls it after its last run; barrier=False
        only when no run was issued, e.g. after a failed setup)."""
        if self._peer_maps:
            import torch.distributed as dist
            torch.cuda.synchronize(self.device)
            if barrier:
                dist.barrier(group=self.group)  # no peer still stores into our buffers
            for ptr, off in self._peer_maps:
                _mom.ipc_close(ptr, off)
            self._peer_maps, self.peers = [], [[], []]

    def _barrier(self, stream):
        if self.comm is not None:
            _mom.nccl_barrier(self.comm, self.barrier_scratch, stream)
        else:  # one-GPU test mode (several ranks on one device, gloo): host barrier
            import torch.distributed as dist
            stream.synchronize()
            dist.barrier(group=self.group)

    def shard_of(self, buf):
        return buf[self.rank * self.S:(self.rank + 1) * self.S]

    # ---------------------------------------------------------------- one prefill request
    def run(self, x, kv_fill=None, compute=None, copy=None, on_layer=None):
        """One GPU: x is [S, d], updated in place to the final layer's input.  Token-sharded: x is
        this rank's [S_local, d] input rows, or a [world * S_local, d] tensor holding them at rows
        rank*S_local (copied into gathered buffer 0 unless x is that buffer).  kv_fill(l, slot)
        writes layer l's stand-in K/V on the current stream.  on_layer(l, buf) is called (host side,
        after enqueueing) before layer l's MLP with the buffer holding layer l's input -- tests use
        it to snapshot teacher-forcing inputs.  Returns a StackResult."""
        compute = compute or torch.cuda.current_stream(self.device)
        copy = copy or torch.cuda.Stream(self.device)
        ev_off = [torch.cuda.Event() for _ in range(self.L)]
        reload_done = []
        reloaded = 0
        h2d = self.h2d

        def reload_layer(j):  # a10 for layer j on the H2D stream, after its D2H completed
            ev = torch.cuda.Event()
            h2d.wait_event(ev_off[j])
            _mom.kv_reload(self.kv_host[j], self.kv_dev[j], h2d, ev)
            reload_done.append(ev)

        launches = 0
        with torch.cuda.stream(compute):
            if self._prev_copies_done is not None:
                compute.wait_event(self._prev_copies_done)
                if h2d is not None:
                    h2d.wait_event(self._prev_copies_done)
            if self.world > 1:
                own = self.shard_of(self.xbuf[0])
                src = x if x.shape[0] == self.S else self.shard_of(x)
                if src.data_ptr() != own.data_ptr():
                    own.copy_(src)
            budget = self.early_budget

            def early_reloads(upto):
                """f4: reload the layers <= upto already offloaded, in order, within the device budget."""
                nonlocal reloaded
                while self.reload and len(reload_done) <= upto and reloaded + self.kv_bytes <= budget:
                    reload_layer(len(reload_done))
                    reloaded += self.kv_bytes

            def offload_layer(l, slot):                                                        # a9
                _mom.kv_offload(slot, self.kv_host[l], compute, copy, ev_off[l])
                early_reloads(l)

            for l in range(self.L):
                if l == self.L - 1 and self.final_layer_release and self.L > 1:
                    budget += self.final_layer_release  # x (but its last row) and the workspace are dead
                    early_reloads(self.L - 2)
                if self.offload:
                    slot = self.kv_ring[l % 2]
                    if l >= 2:
                        compute.wait_event(ev_off[l - 2])   # slot reuse only after its D2H finished
                    if kv_fill is not None:
                        kv_fill(l, slot)
                    # the final layer's D2H is issued after the head: its few hundred us of GEMVs
                    # would otherwise share HBM with the copy engine (-20 % LM-head bandwidth,
                    # profiles/r2_summary.md); the copy itself is the same
                    if l < self.L - 1 or not self.defer_last_offload:
                        offload_layer(l, slot)
                cur = x if self.world == 1 else self.xbuf[gathered_buffer_index(l)]
                if on_layer is not None:
                    on_layer(l, cur)
                wg, wu, wd = self.weights[l]
                if self.folded is not None:
                    wg, wu = self.folded[l]
                if l < self.L - 1:
                    src = x if self.world == 1 else self.shard_of(cur)
                    dst = x if self.world == 1 else self.shard_of(self.xbuf[gathered_buffer_index(l + 1)])
                    if self.folded is not None:                                                    # + f3
                        _mom.mlp_minseq_rmsnorm_fwd(src, wg, wu, wd, dst, self.C, self.norm_eps, self.ws, compute)
                    elif self.world > 1 and self.gather == "fused":                                # a11 fused (f1)
                        _mom.mlp_minseq_fwd_gather(src, src, wg, wu, wd, dst,
                                                   self.peers[gathered_buffer_index(l + 1)], self.C, self.ws, compute)
                    else:
                        _mom.mlp_minseq_fwd(src, src, wg, wu, wd, dst, self.C, self.ws, compute)    # a1-a5
                    if self.world > 1:
                        if self.gather == "fused":
                            self._barrier(compute)
                        else:
                            _mom.allgather_rows(self.xbuf[gathered_buffer_index(l + 1)], self.S, self.comm,
                                                self.rank, self.world, compute)                    # a11 (NCCL)
                    launches += 2 * math.ceil(self.S / self.C)
                elif self.rank == self.owner:
                    last = cur[self.S_total - 1]
                    if self.folded is not None:                                                    # a6 + f3
                        _mom.mlp_last_token_rmsnorm(last, wg, wu, wd, self.y, self.norm_eps, self.ws_last, compute)
                    else:
                        _mom.mlp_last_token(last, last, wg, wu, wd, self.y, self.ws_last, compute)  # a6
                    _mom.lm_head_last(self.y, self.gain, self.eps, self.wh, self.logits, self.argmax,
                                      self.ws_head, compute)                                       # a7-a8
                    launches += 4
            reloaded_before_head = reloaded
            if self.offload and self.defer_last_offload:
                offload_layer(self.L - 1, self.kv_ring[(self.L - 1) % 2])
            x_final = x if self.world == 1 else self.xbuf[gathered_buffer_index(self.L - 1)]
            if self.reload:
                h2d.wait_stream(compute)   # Alg. 1: the rest after the head
                for j in range(len(reload_done), self.L):  # layer order = decode order (f4)
                    reload_layer(j)
                copy.wait_stream(h2d)
            done = torch.cuda.Event()
            done.record(copy)
            self._prev_copies_done = done
            if not self.pipelined_reload:
                compute.wait_stream(copy)
        own = self.rank == self.owner
        return StackResult(self.y if own else None, self.logits if own else None, self.argmax if own else None,
                           self.kv_host, self.kv_dev, launches, reload_done, x_final, copy, reloaded_before_head)
