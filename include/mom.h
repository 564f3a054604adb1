/*
 * mom.h -- C ABI of libmom.so, the B200 (sm_100a) hot path of MOM:
 * "Memory-efficient Offloaded Mini-sequence Inference" (arXiv 2504.12526).
 *
 * Citations: "P:<n>" = line n of the paper text (reference PAPER.md), with its section /
 * algorithm / equation; "S:<n>" = line n of the reference SPEC.md (interfaces only).
 *
 * The path (Alg. 1), per transformer layer, after attention (unchanged):
 *   - offload the layer's K/V to host memory                 -> mom_kv_offload
 *   - non-final layers: partition the MLP input A into M = ceil(S/C) mini-sequences and
 *     compute O_i = MLP(A_i), O = concat(O_i)                 -> mom_mlp_minseq_fwd
 *   - final layer: A_last = A[:, -1, :], O_last = MLP(A_last) -> mom_mlp_last_token
 *     L = LM_Head(O_last), greedy token = argmax L           -> mom_lm_head_last
 *     transfer the offloaded cache back to the GPU            -> mom_kv_reload
 *   - token-sharded multi-GPU: gather every rank's MLP rows   -> mom_allgather_rows
 *
 * MLP is the Llama SwiGLU MLP: MLP(A) = (Swish(A W_gate) (.) A W_up) W_down,
 * Swish(z) = z * sigmoid(z).  Weights are in nn.Linear layout (row-major):
 *   W_gate, W_up: [intermediate, hidden];  W_down: [hidden, intermediate];  W_head: [vocab, hidden].
 * Activations are row-major [rows, hidden] with B = 1 ("we assume B = 1").
 *
 * Conventions (all entry points):
 *   Ownership   The caller allocates every buffer (device memory, pinned host memory,
 *               workspace, streams, events).  The library allocates no memory, keeps no
 *               per-call state, and never synchronises the host.
 *   Async       Compute calls enqueue kernels on `stream` and return.  Kernel faults surface
 *               at the caller's next synchronisation (as with cuBLAS).
 *   Errors      MOM_ERR_INVALID_ARG / _UNSUPPORTED / _WORKSPACE mean NOTHING was enqueued
 *               (arguments are checked before any launch).  MOM_ERR_CUDA / _NCCL report a failed
 *               launch or library call; launches of the same call that preceded it (earlier
 *               mini-sequences) stay enqueued.  mom_last_error() returns a thread-local message.
 *   Tuning      Environment knobs read per call (defaults are the measured best on B200).  Apart
 *               from MOM_GEMV_VARIANT's families (below) none changes results -- outputs are bitwise
 *               identical for every setting (knob tests):
 *               MOM_CTA_GROUP (2)        CTAs per tcgen05 tile (cta_group::2 pair, or 1)
 *               MOM_GROUP_M_A (16), MOM_GROUP_M_B (8)   raster: row blocks per group
 *               MOM_RASTER_B_COLS (0)    phase B by groups of G output-column blocks instead
 *                                        (10 % fewer DRAM reads at G = 8, no measured step gain)
 *               MOM_TMA_POLICY (0)       TMA L2 cache-policy variant of the operand loads
 *               MOM_EPI_L2_HINT (0)      bit 0: H stores evict_first; bit 1: phase-B residual
 *                                        loads / output stores evict_first (measured, no gain)
 *               MOM_FUSED (0)            1: both phases in one persistent launch, grid clamped to
 *                                        cudaOccupancyMaxActiveClusters (phase-B tiles wait on
 *                                        phase-A tiles of other clusters)
 *               MOM_EPI_A_COALESCED (1)  phase-A epilogue through a swizzled smem stage
 *               MOM_MLP_PDL (1)          programmatic dependent launch between the MLP launches
 *               MOM_HALF_TAIL (1)        phase A's last partial wave as half-width tiles
 *               MOM_NB_B (per shape)     phase-B tile width (wave quantisation)
 *               MOM_GATHER_FORWARD (1)   f1: rows of mini-sequence i-1 forwarded during i
 *               MOM_GEMV_PDL (1)         both last-token GEMVs and the argmax reduction PDL-launched
 *               MOM_GEMV_VARIANT (5)     down GEMV: 5 -> each row group K-split over 2 warps (fixed-
 *                                        order combine), 6 -> over 4; loads in flight per row without
 *                                        K-split: 2 -> 8 at 2 blocks/SM, 1 -> 4, 0 -> 2 at 4 blocks/SM;
 *                                        3 -> also gate/up at 4.  5 / 6 sum in their own fixed order
 *                                        (bit-stable per variant; 0-3 are bitwise equal to each other)
 *               MOM_GEMV_PREFETCH (0)    KB of each warp's first W_down rows prefetched to L2
 *               Numerics knob: MOM_FAST_SILU (1: the phase-A SiLU quotient by rcp.approx, <= 2 fp32
 *               ulp; 0: IEEE division, whose per-element slow-path branch serialises the epilogue).
 *   Alignment   Device pointers must be 16-byte aligned and row pitches (hidden*w,
 *               intermediate*w, w = element bytes) multiples of 16 bytes (TMA rule).
 *   Dtypes      MOM_BF16: bf16 storage, fp32 accumulation, fp32 SiLU, one RNE rounding of
 *               the [C, I] intermediate and one of each output (tcgen05 tensor-core path).
 *               MOM_F32: fp32 storage and arithmetic (SIMT path, small parity configs).
 *   Threads     Thread-safe; the only mutable globals are the thread-local error string and
 *               once-initialised per-device caches (SM count, driver entry point).
 *   Streams     mom_stream_t / mom_event_t are cudaStream_t / cudaEvent_t passed as void*.
 */
#ifndef MOM_H_
#define MOM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOM_OK = 0,
  MOM_ERR_INVALID_ARG = 1,  /* null pointer, size < 1, misalignment, bad aliasing, non-pinned host */
  MOM_ERR_UNSUPPORTED = 2,  /* valid arguments this build does not implement (e.g. dtype/shape) */
  MOM_ERR_WORKSPACE = 3,    /* workspace smaller than the matching *_workspace_bytes() query   */
  MOM_ERR_CUDA = 4,         /* a CUDA runtime/driver call failed while enqueueing              */
  MOM_ERR_NCCL = 5          /* NCCL missing or an NCCL call failed                            */
} mom_status_t;

typedef enum { MOM_BF16 = 0, MOM_F32 = 1 } mom_dtype_t;

typedef void *mom_stream_t; /* cudaStream_t (NULL = legacy default stream) */
typedef void *mom_event_t;  /* cudaEvent_t, caller-created                 */

/* Thread-local description of the last non-OK status returned on this thread ("" if none). */
const char *mom_last_error(void);
/* Library version / build string (arch, kernel variants). */
const char *mom_version(void);

/* ------------------------------------------------------------------------------------
 * a1. Mini-sequence plan (host only).  Alg. 1: "Partition A into M = ceil(S/C)
 * mini-sequences {A_i}, where each A_i in R^{B x N x d} and N ~= C"; sizes
 * (C, ..., C, S-(M-1)C).  Writes min(M, cap) (start, length) pairs into
 * starts/lens (either may be NULL when cap == 0) and returns M, or -1 if S < 1 or C < 1.
 * ---------------------------------------------------------------------------------- */
int64_t mom_plan_minseq(int64_t S, int64_t minseq_len, int64_t *starts, int64_t *lens, int64_t cap);

/* ------------------------------------------------------------------------------------
 * a2-a4. Mini-sequence SwiGLU MLP over S tokens.  Alg. 1 P:109-113 with MLP per P:144:
 *   for i = 1..M:  H_i = Swish(A_i W_gate^T) (.) (A_i W_up^T)     [C_i, I]   (Phase A)
 *                  O_i = R_i + H_i W_down^T                        [C_i, d]   (Phase B)
 *   O = concat(O_1..O_M): each O_i is written at its rows of `out` (no concat copy).
 * The [S, I] intermediate of Eq. 1 never exists: only one mini-sequence's H_i
 * lives in `workspace` at a time, so the transient is C*I*w bytes (Eq. 3).
 *
 *   x          device [S, hidden]         MLP input A (the post-attention-norm hidden states)
 *   residual   device [S, hidden] or NULL NULL => out = MLP(x) exactly as Alg. 1's O_i;
 *                                         else out = residual + MLP(x) (fused, fp32 add)
 *   w_gate     device [intermediate, hidden]
 *   w_up       device [intermediate, hidden]
 *   w_down     device [hidden, intermediate]
 *   out        device [S, hidden]         may equal residual and/or x (in place); must not
 *                                         partially overlap either
 *   S, hidden, intermediate >= 1; minseq_len = C >= 1 (C >= S gives M = 1)
 *   workspace  device, >= mom_mlp_minseq_workspace_bytes(S, hidden, intermediate, C, dt)
 * Outputs are bitwise identical for every C (no split-K, no atomics, C-independent tiles).
 * ---------------------------------------------------------------------------------- */
size_t mom_mlp_minseq_workspace_bytes(int64_t S, int64_t hidden, int64_t intermediate,
                                      int64_t minseq_len, mom_dtype_t dt);
mom_status_t mom_mlp_minseq_fwd(const void *x, const void *residual, const void *w_gate,
                                const void *w_up, const void *w_down, void *out, int64_t S,
                                int64_t hidden, int64_t intermediate, int64_t minseq_len,
                                mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                                mom_stream_t stream);

/* The same, with the MLP input in page-locked HOST memory (the end-to-end entry).  For each
 * mini-sequence i the rows of A_i are copied x_host_pinned -> x (device [S, hidden]) on
 * copy_stream, and `stream` waits for exactly those rows before computing O_i, so the PCIe
 * transfer of A_{i+1} overlaps the tensor-core work on A_i (the partition of P:109 applied to
 * the host->device input).
 *   x_free     NULL: copy_stream first waits for all work already queued on `stream` (safe
 *              whatever else reads x).  Else a caller-recorded cudaEvent_t after which nothing
 *              reads or writes x: copy_stream waits on it instead, so the input of the next
 *              request can stream in while `stream` still runs earlier requests (prefetch; the
 *              caller double-buffers x).  A never-recorded event does not delay the copies.
 * residual may equal x (the usual x + MLP(x)).  x_host_pinned must be page-locked (checked);
 * copy_stream must differ from stream.  Other arguments and errors as mom_mlp_minseq_fwd. */
mom_status_t mom_mlp_minseq_fwd_from_host(const void *x_host_pinned, void *x, const void *residual,
                                          const void *w_gate, const void *w_up, const void *w_down,
                                          void *out, int64_t S, int64_t hidden, int64_t intermediate,
                                          int64_t minseq_len, mom_dtype_t dt, void *workspace,
                                          size_t workspace_bytes, mom_stream_t stream,
                                          mom_stream_t copy_stream, mom_event_t x_free);

/* ------------------------------------------------------------------------------------
 * f3. The per-layer RMSNorm folded into the mini-sequence MLP: the Llama
 * block's MLP half  out = x + MLP(RMSNorm(x) (.) g)  (RMSNorm S:126) without
 * writing the normed [S, d] tensor.  Since (RMSNorm(x) (.) g) W^T = r * x (W diag(g))^T with
 * r = 1/sqrt(mean(x^2) + eps) per row:
 *   mom_fold_norm_gain           once per layer: w_folded[j, k] = bf16(w[j, k] * g[k]) for W_gate
 *                                and W_up ([rows, cols] = [I, d]; cols % 8 == 0; may be in place)
 *   mom_mlp_minseq_rmsnorm_fwd   per mini-sequence: r of its rows (one pass over C*d elements),
 *                                then phase A scales the fp32 gate/up accumulators by r before the
 *                                SiLU; phase B adds the residual x.  out may alias x.
 * bf16 only (MOM_ERR_UNSUPPORTED otherwise).  Workspace: one H_i plus C fp32 scales.
 * ---------------------------------------------------------------------------------- */
mom_status_t mom_fold_norm_gain(const void *w, const void *norm_gain, void *w_folded, int64_t rows,
                                int64_t cols, mom_dtype_t dt, mom_stream_t stream);
size_t mom_mlp_minseq_rmsnorm_workspace_bytes(int64_t S, int64_t hidden, int64_t intermediate,
                                              int64_t minseq_len, mom_dtype_t dt);
mom_status_t mom_mlp_minseq_rmsnorm_fwd(const void *x, const void *w_gate_folded,
                                        const void *w_up_folded, const void *w_down, void *out,
                                        int64_t S, int64_t hidden, int64_t intermediate,
                                        int64_t minseq_len, float eps, mom_dtype_t dt,
                                        void *workspace, size_t workspace_bytes, mom_stream_t stream);

/* ------------------------------------------------------------------------------------
 * a6. Final layer on the last token only.  Alg. 1: A_last = A[:, -1, :]
 * (pass x + (S-1)*hidden), O_last = MLP(A_last) (+ residual_last if non-NULL).
 * HBM-bound GEMV pair: h = Swish(W_gate x) (.) (W_up x) kept in fp32 in `workspace`, then
 * out_last = residual_last + W_down h rounded once to dt.
 *   x_last, residual_last (or NULL), out_last: device [hidden]; weights as above.
 *   workspace >= mom_mlp_last_token_workspace_bytes(intermediate).
 * ---------------------------------------------------------------------------------- */
size_t mom_mlp_last_token_workspace_bytes(int64_t intermediate);
mom_status_t mom_mlp_last_token(const void *x_last, const void *residual_last, const void *w_gate,
                                const void *w_up, const void *w_down, void *out_last,
                                int64_t hidden, int64_t intermediate, mom_dtype_t dt,
                                void *workspace, size_t workspace_bytes, mom_stream_t stream);
/* f3 on the last token: out_last = x_last + MLP(RMSNorm(x_last) (.) g) with the gain
 * folded into W_gate / W_up (mom_fold_norm_gain); the gate/up GEMV scales its staged copy of x_last by
 * r = 1/sqrt(mean(x_last^2) + eps) (the sum of squares comes with the staging pass).  eps >= 0; other
 * arguments, workspace and errors as mom_mlp_last_token (residual = x_last; out_last may alias it). */
mom_status_t mom_mlp_last_token_rmsnorm(const void *x_last, const void *w_gate_folded,
                                        const void *w_up_folded, const void *w_down, void *out_last,
                                        int64_t hidden, int64_t intermediate, float eps, mom_dtype_t dt,
                                        void *workspace, size_t workspace_bytes, mom_stream_t stream);

/* ------------------------------------------------------------------------------------
 * a7-a8. LM head on the last token + greedy token.  Alg. 1 P:105 "L = LM_Head(O_last)";
 * the head's intermediate is V.  Optional final RMSNorm prologue (applied
 * after slicing): hn = h / sqrt(mean(h^2) + eps) (.) norm_gain.
 *   h_last     device [hidden] (dtype dt)
 *   norm_gain  device [hidden] (dtype dt) or NULL (no norm; eps ignored)
 *   w_head     device [vocab, hidden] (dtype dt)
 *   logits     device [vocab] fp32, or NULL (not stored)
 *   argmax     device int32[1]: index of the max logit, ties -> lowest index
 *   workspace  >= mom_lm_head_workspace_bytes(vocab)
 * ---------------------------------------------------------------------------------- */
size_t mom_lm_head_workspace_bytes(int64_t vocab);
mom_status_t mom_lm_head_last(const void *h_last, const void *norm_gain, float eps,
                              const void *w_head, float *logits, int32_t *argmax, int64_t hidden,
                              int64_t vocab, mom_dtype_t dt, void *workspace,
                              size_t workspace_bytes, mom_stream_t stream);

/* ------------------------------------------------------------------------------------
 * f2. Vocab-sharded LM head for token-sharded runs: rank r holds W_head rows
 * [vocab_offset, vocab_offset + vocab_shard) and streams only those (1/N of the head's HBM
 * bytes).  mom_lm_head_shard writes the shard's logits (optional) and *best_key, the u64
 * (order-preserving fp32 value << 32 | (2^32-1 - global index)) of its best row; then
 * mom_argmax_allreduce takes the u64 max over ranks (ncclAllReduce, ncclMax; comm == NULL
 * for one rank) and decodes it, so every rank gets the global argmax with ties -> lowest
 * index, bitwise equal to the unsharded mom_lm_head_last.
 *   best_key: device uint64[1], 8-B aligned;  argmax: device int32[1].
 * ---------------------------------------------------------------------------------- */
mom_status_t mom_lm_head_shard(const void *h_last, const void *norm_gain, float eps,
                               const void *w_head_shard, int64_t vocab_offset, int64_t vocab_shard,
                               float *logits_shard, uint64_t *best_key, int64_t hidden,
                               mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                               mom_stream_t stream);
mom_status_t mom_argmax_allreduce(uint64_t *best_key, int32_t *argmax, void *comm, mom_stream_t stream);

/* ------------------------------------------------------------------------------------
 * a9. KV offload.  Alg. 1 P:99 "Update and offload KV cache to CPU"; sec. 3.2 P:127.
 * Records an event on producer_stream, makes copy_stream wait on it, enqueues one
 * cudaMemcpyAsync device->host of `bytes` on copy_stream, then records `done` on
 * copy_stream.  The copy overlaps whatever producer_stream runs next (the MLP).  The
 * caller must not rewrite or free kv_dev before `done` completes.
 *   kv_dev          device, 16-B aligned      kv_host_pinned  page-locked host (checked)
 *   done            caller-created event (may be NULL)
 * a10. KV reload.  Alg. 1 P:106 "Transfer offloaded cache back to GPU for decode stage":
 * one cudaMemcpyAsync host->device on copy_stream, then records `done` (may be NULL).
 * Both: bytes >= 1.  Round trip is bytewise exact.
 * ---------------------------------------------------------------------------------- */
mom_status_t mom_kv_offload(const void *kv_dev, void *kv_host_pinned, size_t bytes,
                            mom_stream_t producer_stream, mom_stream_t copy_stream,
                            mom_event_t done);
mom_status_t mom_kv_reload(const void *kv_host_pinned, void *kv_dev, size_t bytes,
                           mom_stream_t copy_stream, mom_event_t done);

/* ------------------------------------------------------------------------------------
 * a11. Token-sharded multi-GPU (one process per GPU).  The S tokens are split into
 * contiguous row ranges per rank; the position-wise MLP needs no exchange, and one
 * in-place all-gather per layer rebuilds the [S, hidden] rows the next (unchanged,
 * P:81) attention layer needs.  NCCL is loaded at run time (dlopen libnccl.so.2).
 *   mom_nccl_get_unique_id   rank 0 writes the 128-byte NCCL unique id to id_out
 *   mom_nccl_comm_init       every rank: *comm_out = ncclCommInitRank(nranks, id, rank)
 *                            (the current CUDA device must already be set)
 *   mom_nccl_comm_destroy    ncclCommDestroy
 *   mom_allgather_rows       rows: device [nranks * rows_per_rank, hidden]; this rank's
 *                            shard is at row rank*rows_per_rank; in-place ncclAllGather on
 *                            `stream`; after completion every rank holds all rows.
 * ---------------------------------------------------------------------------------- */
mom_status_t mom_nccl_barrier(void *comm, int32_t *scratch /* device int32[1] */, mom_stream_t stream);

/* f1: the all-gather fused into the down-GEMM epilogue.  Same as
 * mom_mlp_minseq_fwd, and every output row O_i is ALSO stored, from the phase-B epilogue
 * that produces it, into each of the n_peers buffers peer_out[k] (same row offsets as `out`):
 * the peers' gathered [N*S_local, hidden] buffers at this rank's shard, NVLink-mapped with
 * mom_ipc_open_handle.  The rows cross NVLink while the tensor cores keep working, instead
 * of in a separate collective after the layer.  After the call, one mom_nccl_barrier on
 * the same stream guarantees that every rank's peer stores of THIS call have landed before any
 * rank runs past the barrier.  It does not protect a reader of the destination rows from the
 * stores of a LATER call: a caller whose ranks read the gathered rows while the next layer runs
 * (a full model's attention over all rows) must alternate two gathered buffers, layer l writing
 * buffer (l+1) % 2 -- then the barrier of layer l, which every rank passes only after its own
 * layer-l work, orders all reads of a buffer before the next stores into it (stack.py does this).
 *   0 <= n_peers <= 7; peer_out[k] 16-B aligned; bf16 only when n_peers > 0.
 * IPC plumbing: mom_ipc_get_handle returns the 64-byte cudaIpcMemHandle of the allocation
 * holding dev_ptr and dev_ptr's offset in it (torch sub-allocates); mom_ipc_open_handle maps
 * a peer's handle (cudaIpcMemLazyEnablePeerAccess) and returns base + offset;
 * mom_ipc_close unmaps it. */
mom_status_t mom_mlp_minseq_fwd_gather(const void *x, const void *residual, const void *w_gate,
                                       const void *w_up, const void *w_down, void *out,
                                       void *const *peer_out, int n_peers, int64_t S, int64_t hidden,
                                       int64_t intermediate, int64_t minseq_len, mom_dtype_t dt,
                                       void *workspace, size_t workspace_bytes, mom_stream_t stream);
/* The end-to-end entry of token-sharded runs: mom_mlp_minseq_fwd_from_host (input streamed from
 * pinned host memory per mini-sequence, optional x_free prefetch) whose output rows also go to
 * the n_peers buffers as in mom_mlp_minseq_fwd_gather.  Arguments and errors as those two. */
mom_status_t mom_mlp_minseq_fwd_from_host_gather(const void *x_host_pinned, void *x, const void *residual,
                                                 const void *w_gate, const void *w_up, const void *w_down,
                                                 void *out, void *const *peer_out, int n_peers, int64_t S,
                                                 int64_t hidden, int64_t intermediate, int64_t minseq_len,
                                                 mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                                                 mom_stream_t stream, mom_stream_t copy_stream,
                                                 mom_event_t x_free);
mom_status_t mom_ipc_get_handle(const void *dev_ptr, void *handle_out /* 64 B */, int64_t *offset_out);
mom_status_t mom_ipc_open_handle(const void *handle /* 64 B */, int64_t offset, void **dev_ptr_out);
mom_status_t mom_ipc_close(void *dev_ptr, int64_t offset);

mom_status_t mom_nccl_get_unique_id(void *id_out /* 128 bytes */);
mom_status_t mom_nccl_comm_init(void **comm_out, int nranks, const void *id /* 128 B */, int rank);
mom_status_t mom_nccl_comm_destroy(void *comm);
/* Failure detection.  Every NCCL-issuing entry (mom_allgather_rows, mom_nccl_barrier,
 * mom_argmax_allreduce) polls ncclCommGetAsyncError after enqueueing and returns MOM_ERR_NCCL if the
 * communicator is in an error state (a failed or aborted peer, an error inside an earlier collective).
 *   mom_nccl_check        the same poll, host-side and non-blocking: a caller waiting on a stream that
 *                         holds collectives calls it periodically; MOM_OK while healthy
 *                         (ncclSuccess / ncclInProgress), MOM_ERR_NCCL with the NCCL reason otherwise.
 *   mom_nccl_comm_count   *nranks_out = ncclCommCount(comm) (confirms the world size after init).
 *   mom_nccl_comm_abort   ncclCommAbort: unblocks collectives stuck on a dead peer; the comm is freed. */
mom_status_t mom_nccl_check(void *comm);
mom_status_t mom_nccl_comm_count(void *comm, int *nranks_out);
mom_status_t mom_nccl_comm_abort(void *comm);
mom_status_t mom_allgather_rows(void *rows, int64_t rows_per_rank, int64_t hidden, mom_dtype_t dt,
                                void *comm, int rank, int nranks, mom_stream_t stream);

/* ------------------------------------------------------------------------------------
 * Instrumentation (used by bench.py for the per-kernel roofline; not part of the path).
 * While enabled on the calling thread, every kernel launch issued by the compute entry
 * points is bracketed by cudaEventRecord(events[2j]) / cudaEventRecord(events[2j+1]) on its
 * stream, kinds[j] is set to the launch kind and *count is incremented (j = *count before
 * the launch; launches beyond `capacity` pairs are not recorded).  Kinds:
 *   0 phase A tcgen05 (gate/up + SiLU*mul)   1 phase B tcgen05 (down + residual)
 *   2 phase A fp32 SIMT                      3 phase B fp32 SIMT
 *   4 last-token GEMV pair                   5 LM head GEMV + argmax
 * events: caller-created cudaEvent_t array of 2*capacity; kinds: int32[capacity];
 * count: host int64.  Pass events == NULL to disable.  Thread-local, host-side only.
 * ---------------------------------------------------------------------------------- */
mom_status_t mom_set_timing_events(mom_event_t *events, int32_t *kinds, int64_t capacity, int64_t *count);

/* In-kernel trace (tools/kernel_trace.py; not part of the path).  While enabled on the calling
 * thread, the j-th tcgen05 MLP launch (j = *count before it, j < capacity) writes stamps to
 * dev_buf[(j * 160 + cta) * 8 + k]: %globaltimer (ns) at k = 0 CTA entry, 1 first MMA issued and
 * 2 last MMA issued (leader CTAs), 3 CTA exit; the SM's clock64 at k = 4 first and 5 last MMA
 * (so the SM clock over the launch is (k5 - k4) / (k2 - k1)); k = 6 the SM cycles epilogue warp 4
 * spent in tile epilogues (summed), k = 7 their count; *count is incremented per launch.
 * dev_buf: device uint64[capacity * 160 * 8], zeroed by the caller.  NULL disables.  A launch whose
 * persistent grid exceeds 160 CTAs (a part with more than 160 SMs) is not traced (no slot used). */
mom_status_t mom_set_kernel_trace(void *dev_buf, int64_t capacity, int64_t *count);

#ifdef __cplusplus
} /* extern "C" */
#endif
#endif /* MOM_H_ */
