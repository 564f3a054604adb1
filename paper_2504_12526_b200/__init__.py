"""B200-native hot path of MOM (arXiv 2504.12526): the mini-sequence prefill MLP.

The product is ``libmom.so`` (C ABI, ``include/mom.h``), hand-written sm_100a kernels:
tcgen05/TMEM/TMA SwiGLU MLP per mini-sequence, HBM-streaming last-token GEMVs with argmax,
KV offload/reload on a side stream, NCCL all-gather for token-sharded runs.  This package
is the thin ctypes binding (same names as the C entry points, ``mom_`` prefix dropped).
"""
from ._mom import (  # noqa: F401
    LIB_PATH,
    LaunchTimer,
    MomError,
    allgather_rows,
    argmax_allreduce,
    lm_head_shard,
    kv_offload,
    kv_reload,
    lib,
    lm_head_last,
    mlp_last_token,
    fold_norm_gain,
    ipc_close,
    ipc_get_handle,
    ipc_open_handle,
    mlp_minseq_fwd,
    mlp_minseq_fwd_from_host,
    mlp_minseq_fwd_gather,
    mlp_minseq_rmsnorm_fwd,
    mlp_minseq_workspace_bytes,
    nccl_comm_destroy,
    nccl_barrier,
    nccl_comm_init,
    nccl_get_unique_id,
    plan_minseq,
    version,
)
