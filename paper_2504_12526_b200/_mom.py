"""Thin ctypes binding of libmom.so (include/mom.h).  Argument marshalling only: every step
of the path runs in the library's CUDA kernels; torch supplies device memory, pinned host
memory and streams.  There is no fallback: if libmom.so is missing or a call fails, an
exception is raised."""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libmom.so")

MOM_OK, MOM_ERR_INVALID_ARG, MOM_ERR_UNSUPPORTED, MOM_ERR_WORKSPACE, MOM_ERR_CUDA, MOM_ERR_NCCL = range(6)
MOM_BF16, MOM_F32 = 0, 1
STATUS_NAMES = {0: "MOM_OK", 1: "MOM_ERR_INVALID_ARG", 2: "MOM_ERR_UNSUPPORTED", 3: "MOM_ERR_WORKSPACE",
                4: "MOM_ERR_CUDA", 5: "MOM_ERR_NCCL"}

# name -> (restype, argtypes); the symbol table checked by tests/test_abi.py against include/mom.h
_p, _i64, _i32, _sz, _f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.c_float
SIGNATURES = {
    "mom_last_error": (ctypes.c_char_p, []),
    "mom_version": (ctypes.c_char_p, []),
    "mom_plan_minseq": (_i64, [_i64, _i64, _p, _p, _i64]),
    "mom_mlp_minseq_workspace_bytes": (_sz, [_i64, _i64, _i64, _i64, _i32]),
    "mom_mlp_minseq_fwd": (_i32, [_p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i32, _p, _sz, _p]),
    "mom_mlp_minseq_fwd_from_host": (_i32, [_p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i32, _p, _sz, _p,
                                            _p, _p]),
    "mom_fold_norm_gain": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p]),
    "mom_mlp_minseq_rmsnorm_workspace_bytes": (_sz, [_i64, _i64, _i64, _i64, _i32]),
    "mom_mlp_minseq_rmsnorm_fwd": (_i32, [_p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _f32, _i32, _p, _sz, _p]),
    "mom_mlp_last_token_workspace_bytes": (_sz, [_i64]),
    "mom_mlp_last_token": (_i32, [_p, _p, _p, _p, _p, _p, _i64, _i64, _i32, _p, _sz, _p]),
    "mom_mlp_last_token_rmsnorm": (_i32, [_p, _p, _p, _p, _p, _i64, _i64, _f32, _i32, _p, _sz, _p]),
    "mom_lm_head_workspace_bytes": (_sz, [_i64]),
    "mom_lm_head_last": (_i32, [_p, _p, _f32, _p, _p, _p, _i64, _i64, _i32, _p, _sz, _p]),
    "mom_lm_head_shard": (_i32, [_p, _p, _f32, _p, _i64, _i64, _p, _p, _i64, _i32, _p, _sz, _p]),
    "mom_argmax_allreduce": (_i32, [_p, _p, _p, _p]),
    "mom_kv_offload": (_i32, [_p, _p, _sz, _p, _p, _p]),
    "mom_kv_reload": (_i32, [_p, _p, _sz, _p, _p]),
    "mom_nccl_get_unique_id": (_i32, [_p]),
    "mom_nccl_comm_init": (_i32, [ctypes.POINTER(ctypes.c_void_p), _i32, _p, _i32]),
    "mom_nccl_comm_destroy": (_i32, [_p]),
    "mom_nccl_check": (_i32, [_p]),
    "mom_nccl_comm_count": (_i32, [_p, ctypes.POINTER(ctypes.c_int)]),
    "mom_nccl_comm_abort": (_i32, [_p]),
    "mom_allgather_rows": (_i32, [_p, _i64, _i64, _i32, _p, _i32, _i32, _p]),
    "mom_set_timing_events": (_i32, [_p, _p, _i64, _p]),
    "mom_set_kernel_trace": (_i32, [_p, _i64, ctypes.POINTER(ctypes.c_int64)]),
    "mom_nccl_barrier": (_i32, [_p, _p, _p]),
    "mom_mlp_minseq_fwd_gather": (_i32, [_p, _p, _p, _p, _p, _p, _p, _i32, _i64, _i64, _i64, _i64, _i32, _p, _sz,
                                         _p]),
    "mom_mlp_minseq_fwd_from_host_gather": (_i32, [_p, _p, _p, _p, _p, _p, _p, _p, _i32, _i64, _i64, _i64, _i64,
                                                   _i32, _p, _sz, _p, _p, _p]),
    "mom_ipc_get_handle": (_i32, [_p, _p, ctypes.POINTER(ctypes.c_int64)]),
    "mom_ipc_open_handle": (_i32, [_p, _i64, ctypes.POINTER(ctypes.c_void_p)]),
    "mom_ipc_close": (_i32, [_p, _i64]),
}

KIND_NAMES = {0: "phaseA_tc", 1: "phaseB_tc", 2: "phaseA_f32", 3: "phaseB_f32", 4: "last_token_gemv",
              5: "lm_head_gemv", 6: "mlp_fused_tc"}
KERNELS_PER_KIND = {4: 2, 5: 2}  # the GEMV kinds launch two kernels each (plus 1 for the others)


class LaunchTimer:
    """Per-launch CUDA-event timing of the library's kernels (mom_set_timing_events).
    Events are recorded by the library on the stream each kernel is launched on."""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(2 * capacity)]
        for e in self.events:  # force creation of the underlying cudaEvent_t
            e.record()
        torch.cuda.synchronize()
        self._handles = (ctypes.c_void_p * (2 * capacity))(*[e.cuda_event for e in self.events])
        self._kinds = (ctypes.c_int32 * capacity)()
        self._count = ctypes.c_int64(0)

    def __enter__(self):
        self._count.value = 0
        _check(lib().mom_set_timing_events(self._handles, self._kinds, self.capacity, ctypes.byref(self._count)))
        return self

    def __exit__(self, *exc):
        lib().mom_set_timing_events(None, None, 0, None)
        return False

    def results(self):
        """[(kind_name, ms)] for every recorded launch (call after synchronising)."""
        out = []
        for j in range(min(self._count.value, self.capacity)):
            out.append((KIND_NAMES.get(self._kinds[j], str(self._kinds[j])),
                        self.events[2 * j].elapsed_time(self.events[2 * j + 1])))
        return out

    def timeline(self, origin):
        """[(kind_name, start_ms, end_ms)] relative to the torch.cuda.Event `origin` (recorded on
        the same stream before the launches); shows the gaps between launches."""
        out = []
        for j in range(min(self._count.value, self.capacity)):
            out.append((KIND_NAMES.get(self._kinds[j], str(self._kinds[j])),
                        origin.elapsed_time(self.events[2 * j]), origin.elapsed_time(self.events[2 * j + 1])))
        return out


_lib = None


class MomError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libmom.so (raises if it was not built -- there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2504_12526_b200.build` "
                              "or __graft_entry__.build()")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def _check(status: int):
    if status != MOM_OK:
        raise MomError(status, lib().mom_last_error().decode(errors="replace"))


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return MOM_BF16
    if t.dtype == torch.float32:
        return MOM_F32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _ptr(t):
    """Raw pointer of a tensor argument.  The C ABI takes dense row-major buffers: a strided view
    (e.g. a transposed weight) would be read with the wrong layout, so it is rejected here."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if not t.is_contiguous():
        raise ValueError(f"libmom takes contiguous row-major tensors (got shape {tuple(t.shape)}, "
                         f"stride {tuple(t.stride())})")
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _event_handle(done):
    if done is None:
        return None
    return done.cuda_event or None


def version() -> str:
    return lib().mom_version().decode()


def plan_minseq(S: int, minseq_len: int):
    """Alg. 1: [(start, length)] of the M = ceil(S/C) mini-sequences (host only)."""
    M = lib().mom_plan_minseq(S, minseq_len, None, None, 0)
    if M < 0:
        raise ValueError("S and minseq_len must be >= 1")
    starts = (ctypes.c_int64 * M)()
    lens = (ctypes.c_int64 * M)()
    lib().mom_plan_minseq(S, minseq_len, starts, lens, M)
    return [(starts[i], lens[i]) for i in range(M)]


def mlp_minseq_workspace_bytes(S: int, hidden: int, intermediate: int, minseq_len: int, dtype) -> int:
    dt = MOM_BF16 if dtype == torch.bfloat16 else MOM_F32
    return int(lib().mom_mlp_minseq_workspace_bytes(S, hidden, intermediate, minseq_len, dt))


def _expect(name, t, shape, dtype):
    if t is None:
        return
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype:
        raise ValueError(f"{name}: expected shape {tuple(shape)} dtype {dtype}, got {tuple(t.shape)} {t.dtype}")


def _check_mlp(x, residual, w_gate, w_up, w_down, out, x_host=None):
    """Shapes of the MLP arguments (the C ABI trusts the sizes it is given): x, residual, out, x_host
    [S, d]; W_gate, W_up [I, d]; W_down [d, I]; one dtype."""
    if x.dim() != 2 or w_gate.dim() != 2:
        raise ValueError("x and w_gate must be 2-D")
    (S, d), I = x.shape, w_gate.shape[0]
    for name, t, shape in (("residual", residual, (S, d)), ("w_gate", w_gate, (I, d)), ("w_up", w_up, (I, d)),
                           ("w_down", w_down, (d, I)), ("out", out, (S, d)), ("x_host", x_host, (S, d))):
        _expect(name, t, shape, x.dtype)


def _check_gemv(x, residual, w_gate, w_up, w_down, out):
    d, I = x.shape[-1], w_gate.shape[0]
    for name, t, shape in (("x_last", x, (d,)), ("residual_last", residual, (d,)), ("w_gate", w_gate, (I, d)),
                           ("w_up", w_up, (I, d)), ("w_down", w_down, (d, I)), ("out_last", out, (d,))):
        _expect(name, t, shape, x.dtype)


def mlp_minseq_fwd(x, residual, w_gate, w_up, w_down, out, minseq_len: int, workspace=None, stream=None):
    """Alg. 1: out = residual + concat_i MLP(x_i) over M = ceil(S/C) mini-sequences."""
    _check_mlp(x, residual, w_gate, w_up, w_down, out)
    S, hidden = x.shape
    I = w_gate.shape[0]
    dt = _dt(x)
    if workspace is None:
        nbytes = lib().mom_mlp_minseq_workspace_bytes(S, hidden, I, minseq_len, dt)
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().mom_mlp_minseq_fwd(_ptr(x), _ptr(residual), _ptr(w_gate), _ptr(w_up), _ptr(w_down), _ptr(out),
                                    S, hidden, I, minseq_len, dt, _ptr(workspace), ws_bytes, _stream(stream)))
    return out


def mlp_minseq_fwd_from_host(x_host, x, residual, w_gate, w_up, w_down, out, minseq_len: int, workspace=None,
                             stream=None, copy_stream=None, x_free=None):
    """End-to-end entry: x_host (pinned) is streamed into x one mini-sequence at a time on
    copy_stream while the MLP of the previous mini-sequence runs on stream.  x_free: optional
    torch.cuda.Event after which x is free (the copies wait on it instead of on `stream`)."""
    _check_mlp(x, residual, w_gate, w_up, w_down, out, x_host)
    S, hidden = x.shape
    I = w_gate.shape[0]
    dt = _dt(x)
    if workspace is None:
        nbytes = lib().mom_mlp_minseq_workspace_bytes(S, hidden, I, minseq_len, dt)
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    if copy_stream is None:
        raise ValueError("copy_stream is required")
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().mom_mlp_minseq_fwd_from_host(_ptr(x_host), _ptr(x), _ptr(residual), _ptr(w_gate), _ptr(w_up),
                                              _ptr(w_down), _ptr(out), S, hidden, I, minseq_len, dt, _ptr(workspace),
                                              ws_bytes, _stream(stream), _stream(copy_stream),
                                              _event_handle(x_free)))
    return out


def fold_norm_gain(w, norm_gain, w_folded=None, stream=None):
    """f3: w_folded = w * diag(norm_gain) (bf16), once per layer for W_gate and W_up."""
    w_folded = torch.empty_like(w) if w_folded is None else w_folded
    rows, cols = w.shape
    _check(lib().mom_fold_norm_gain(_ptr(w), _ptr(norm_gain), _ptr(w_folded), rows, cols, _dt(w), _stream(stream)))
    return w_folded


def mlp_minseq_rmsnorm_fwd(x, w_gate_folded, w_up_folded, w_down, out, minseq_len: int, eps: float,
                           workspace=None, stream=None):
    """f3: out = x + MLP(RMSNorm(x) * g) with g folded into W_gate/W_up, per mini-sequence."""
    _check_mlp(x, None, w_gate_folded, w_up_folded, w_down, out)
    S, hidden = x.shape
    I = w_gate_folded.shape[0]
    dt = _dt(x)
    if workspace is None:
        nbytes = lib().mom_mlp_minseq_rmsnorm_workspace_bytes(S, hidden, I, minseq_len, dt)
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    _check(lib().mom_mlp_minseq_rmsnorm_fwd(_ptr(x), _ptr(w_gate_folded), _ptr(w_up_folded), _ptr(w_down), _ptr(out),
                                            S, hidden, I, minseq_len, float(eps), dt, _ptr(workspace),
                                            workspace.numel() * workspace.element_size(), _stream(stream)))
    return out


def mlp_last_token(x_last, residual_last, w_gate, w_up, w_down, out_last, workspace=None, stream=None):
    """Alg. 1: O_last = residual_last + MLP(A_last) on one token (GEMV pair)."""
    _check_gemv(x_last, residual_last, w_gate, w_up, w_down, out_last)
    hidden = x_last.shape[-1]
    I = w_gate.shape[0]
    dt = _dt(x_last)
    if workspace is None:
        workspace = torch.empty(lib().mom_mlp_last_token_workspace_bytes(I), dtype=torch.uint8, device=x_last.device)
    _check(lib().mom_mlp_last_token(_ptr(x_last), _ptr(residual_last), _ptr(w_gate), _ptr(w_up), _ptr(w_down),
                                    _ptr(out_last), hidden, I, dt, _ptr(workspace),
                                    workspace.numel() * workspace.element_size(), _stream(stream)))
    return out_last


def mlp_last_token_rmsnorm(x_last, w_gate_folded, w_up_folded, w_down, out_last, eps: float, workspace=None,
                           stream=None):
    """f3 on the last token: out_last = x_last + MLP(RMSNorm(x_last) * g), g folded into W_gate/W_up."""
    _check_gemv(x_last, None, w_gate_folded, w_up_folded, w_down, out_last)
    hidden = x_last.shape[-1]
    I = w_gate_folded.shape[0]
    dt = _dt(x_last)
    if workspace is None:
        workspace = torch.empty(lib().mom_mlp_last_token_workspace_bytes(I), dtype=torch.uint8, device=x_last.device)
    _check(lib().mom_mlp_last_token_rmsnorm(_ptr(x_last), _ptr(w_gate_folded), _ptr(w_up_folded), _ptr(w_down),
                                            _ptr(out_last), hidden, I, float(eps), dt, _ptr(workspace),
                                            workspace.numel() * workspace.element_size(), _stream(stream)))
    return out_last


def lm_head_last(h_last, norm_gain, eps: float, w_head, logits, argmax, workspace=None, stream=None):
    """Alg. 1: logits = W_head . rmsnorm(h_last) (fp32) and argmax (int32, ties -> lowest)."""
    hidden = h_last.shape[-1]
    V = w_head.shape[0]
    _expect("h_last", h_last, (hidden,), h_last.dtype)
    _expect("norm_gain", norm_gain, (hidden,), h_last.dtype)
    _expect("w_head", w_head, (V, hidden), h_last.dtype)
    _expect("logits", logits, (V,), torch.float32)
    _expect("argmax", argmax, (1,), torch.int32)
    dt = _dt(h_last)
    if workspace is None:
        workspace = torch.empty(lib().mom_lm_head_workspace_bytes(V), dtype=torch.uint8, device=h_last.device)
    _check(lib().mom_lm_head_last(_ptr(h_last), _ptr(norm_gain), float(eps), _ptr(w_head), _ptr(logits),
                                  _ptr(argmax), hidden, V, dt, _ptr(workspace),
                                  workspace.numel() * workspace.element_size(), _stream(stream)))
    return argmax


def lm_head_shard(h_last, norm_gain, eps: float, w_head_shard, vocab_offset: int, logits_shard, best_key,
                  workspace=None, stream=None):
    """f2: this rank's vocab shard of the LM head; best_key (device int64[1]) gets the packed best."""
    hidden = h_last.shape[-1]
    Vs = w_head_shard.shape[0]
    _expect("h_last", h_last, (hidden,), h_last.dtype)
    _expect("norm_gain", norm_gain, (hidden,), h_last.dtype)
    _expect("w_head_shard", w_head_shard, (Vs, hidden), h_last.dtype)
    _expect("logits_shard", logits_shard, (Vs,), torch.float32)
    _expect("best_key", best_key, (1,), torch.int64)
    if workspace is None:
        workspace = torch.empty(lib().mom_lm_head_workspace_bytes(Vs), dtype=torch.uint8, device=h_last.device)
    _check(lib().mom_lm_head_shard(_ptr(h_last), _ptr(norm_gain), float(eps), _ptr(w_head_shard), vocab_offset, Vs,
                                   _ptr(logits_shard), _ptr(best_key), hidden, _dt(h_last), _ptr(workspace),
                                   workspace.numel() * workspace.element_size(), _stream(stream)))
    return best_key


def argmax_allreduce(best_key, argmax, comm=None, stream=None):
    """f2: u64 max of best_key over ranks (NCCL; comm None = one rank), decoded into argmax."""
    _check(lib().mom_argmax_allreduce(_ptr(best_key), _ptr(argmax), comm, _stream(stream)))
    return argmax


def _copy_bytes(kv_dev, kv_host, nbytes, what) -> int:
    """Bytes of a KV copy: nbytes (default: all of kv_dev); both buffers must hold at least that."""
    dev_b = kv_dev.numel() * kv_dev.element_size()
    host_b = kv_host.numel() * kv_host.element_size()
    n = dev_b if nbytes is None else int(nbytes)
    if n < 0 or n > dev_b or n > host_b:
        raise ValueError(f"{what}: {n} bytes requested, device buffer {dev_b} B, host buffer {host_b} B")
    return n


def kv_offload(kv_dev, kv_host_pinned, producer_stream=None, copy_stream=None, done=None, nbytes=None):
    """Alg. 1: async D2H of one layer's K/V into pinned host memory on copy_stream."""
    n = _copy_bytes(kv_dev, kv_host_pinned, nbytes, "kv_offload")
    ev = _event_handle(done)
    _check(lib().mom_kv_offload(_ptr(kv_dev), _ptr(kv_host_pinned), n, _stream(producer_stream),
                                _stream(copy_stream), ev))
    if done is not None and ev is None:  # torch creates its event lazily: record after the copy
        done.record(copy_stream if copy_stream is not None else torch.cuda.current_stream())
    return done


def kv_reload(kv_host_pinned, kv_dev, copy_stream=None, done=None, nbytes=None):
    """Alg. 1: async H2D of the offloaded cache before decode."""
    n = _copy_bytes(kv_dev, kv_host_pinned, nbytes, "kv_reload")
    ev = _event_handle(done)
    _check(lib().mom_kv_reload(_ptr(kv_host_pinned), _ptr(kv_dev), n, _stream(copy_stream), ev))
    if done is not None and ev is None:
        done.record(copy_stream if copy_stream is not None else torch.cuda.current_stream())
    return done


def mlp_minseq_fwd_gather(x, residual, w_gate, w_up, w_down, out, peer_out, minseq_len: int, workspace=None,
                          stream=None):
    """f1: mlp_minseq_fwd whose phase-B epilogue also stores every output row into each peer
    buffer (device pointers, e.g. from ipc_open_handle, offset like `out`)."""
    _check_mlp(x, residual, w_gate, w_up, w_down, out)
    S, hidden = x.shape
    I = w_gate.shape[0]
    dt = _dt(x)
    if workspace is None:
        nbytes = lib().mom_mlp_minseq_workspace_bytes(S, hidden, I, minseq_len, dt)
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    peers = [_ptr(p) for p in peer_out]
    arr = (ctypes.c_void_p * max(1, len(peers)))(*peers)
    _check(lib().mom_mlp_minseq_fwd_gather(_ptr(x), _ptr(residual), _ptr(w_gate), _ptr(w_up), _ptr(w_down), _ptr(out),
                                           arr, len(peers), S, hidden, I, minseq_len, dt, _ptr(workspace),
                                           workspace.numel() * workspace.element_size(), _stream(stream)))
    return out


def mlp_minseq_fwd_from_host_gather(x_host, x, residual, w_gate, w_up, w_down, out, peer_out, minseq_len: int,
                                    workspace=None, stream=None, copy_stream=None, x_free=None):
    """End-to-end entry of token-sharded runs: mlp_minseq_fwd_from_host whose output rows also go
    to every peer buffer (as mlp_minseq_fwd_gather)."""
    _check_mlp(x, residual, w_gate, w_up, w_down, out, x_host)
    S, hidden = x.shape
    I = w_gate.shape[0]
    dt = _dt(x)
    if workspace is None:
        nbytes = lib().mom_mlp_minseq_workspace_bytes(S, hidden, I, minseq_len, dt)
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    if copy_stream is None:
        raise ValueError("copy_stream is required")
    peers = [_ptr(p) for p in peer_out]
    arr = (ctypes.c_void_p * max(1, len(peers)))(*peers)
    _check(lib().mom_mlp_minseq_fwd_from_host_gather(
        _ptr(x_host), _ptr(x), _ptr(residual), _ptr(w_gate), _ptr(w_up), _ptr(w_down), _ptr(out), arr, len(peers),
        S, hidden, I, minseq_len, dt, _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream),
        _stream(copy_stream), _event_handle(x_free)))
    return out


def ipc_get_handle(t) -> tuple[bytes, int]:
    """(64-byte cudaIpcMemHandle of t's allocation, byte offset of t in it)."""
    buf = (ctypes.c_uint8 * 64)()
    off = ctypes.c_int64(0)
    _check(lib().mom_ipc_get_handle(_ptr(t), buf, ctypes.byref(off)))
    return bytes(buf), off.value


def ipc_open_handle(handle: bytes, offset: int) -> int:
    buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    ptr = ctypes.c_void_p()
    _check(lib().mom_ipc_open_handle(buf, offset, ctypes.byref(ptr)))
    return ptr.value


def ipc_close(ptr: int, offset: int):
    _check(lib().mom_ipc_close(ptr, offset))


def nccl_barrier(comm: int, scratch, stream=None):
    _check(lib().mom_nccl_barrier(comm, _ptr(scratch), _stream(stream)))


def nccl_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().mom_nccl_get_unique_id(buf))
    return bytes(buf)


def nccl_comm_init(nranks: int, uid: bytes, rank: int) -> int:
    comm = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(lib().mom_nccl_comm_init(ctypes.byref(comm), nranks, buf, rank))
    return comm.value


def nccl_comm_destroy(comm: int):
    _check(lib().mom_nccl_comm_destroy(comm))


def nccl_check(comm: int):
    """Raises MomError(MOM_ERR_NCCL) if the communicator is in an error state (non-blocking poll)."""
    _check(lib().mom_nccl_check(comm))


def nccl_comm_count(comm: int) -> int:
    n = ctypes.c_int(0)
    _check(lib().mom_nccl_comm_count(comm, ctypes.byref(n)))
    return n.value


def nccl_comm_abort(comm: int):
    _check(lib().mom_nccl_comm_abort(comm))


def allgather_rows(rows, rows_per_rank: int, comm: int, rank: int, nranks: int, stream=None):
    """In-place all-gather of every rank's [rows_per_rank, hidden] shard of `rows`."""
    hidden = rows.shape[-1]
    if rows.dim() != 2 or rows.shape[0] < nranks * rows_per_rank:
        raise ValueError(f"allgather_rows: rows must be [>= {nranks} * {rows_per_rank}, hidden], "
                         f"got {tuple(rows.shape)}")
    _check(lib().mom_allgather_rows(_ptr(rows), rows_per_rank, hidden, _dt(rows), comm, rank, nranks,
                                    _stream(stream)))
    return rows
