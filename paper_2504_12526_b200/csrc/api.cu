// api.cu -- the C ABI of libmom.so (include/mom.h): argument validation, mini-sequence
// planning (Alg. 1), TMA descriptor encoding, kernel launches, KV offload/reload
// (sec. 3.2) and the NCCL all-gather for token-sharded runs.
#include <nvtx3/nvToolsExt.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/mom.h"
#include "kernels.h"

namespace {

thread_local char g_err[512] = "";

mom_status_t fail(mom_status_t st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

mom_status_t cuda_fail(cudaError_t e, const char *what) {
  return fail(MOM_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t dtype_bytes(mom_dtype_t dt) { return dt == MOM_BF16 ? 2 : 4; }

bool valid_dtype(mom_dtype_t dt) { return dt == MOM_BF16 || dt == MOM_F32; }

// [a, a+na) and [b, b+nb) overlap but are not identical
bool partial_overlap(const void *a, size_t na, const void *b, size_t nb) {
  if (!a || !b) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  if (a0 == b0) return false;
  return a0 < b0 + nb && b0 < a0 + na;
}

// ---- per-device cache: SM count (B200: 148) ----
int num_sms_current(int *out) {
  static std::mutex mu;
  static int cache[64];
  static bool have[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && have[dev]) {
    *out = cache[dev];
    return 0;
  }
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (dev < 64) {
    cache[dev] = n;
    have[dev] = true;
  }
  *out = n;
  return 0;
}

// ---- cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda) ----
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static std::once_flag once;
  static EncodeFn fn = nullptr;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2D bf16 row-major [rows, cols] tensor, box = 64 columns (128 B, one 128-B swizzle span) x 128 rows.
mom_status_t make_tmap(CUtensorMap *m, const void *base, uint64_t rows, uint64_t cols, const char *what,
                       uint32_t box_rows = 128) {
  EncodeFn enc = encode_fn();
  if (!enc) return fail(MOM_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MOM_ERR_CUDA, "cuTensorMapEncodeTiled(%s) failed: %d", what, (int)r);
  return MOM_OK;
}

// ---- per-thread launch timing hook (mom_set_timing_events) ----
struct TimingHook {
  cudaEvent_t *ev = nullptr;
  int32_t *kinds = nullptr;
  int64_t cap = 0;
  int64_t *count = nullptr;
};
thread_local TimingHook g_hook;

// ---- per-thread in-kernel trace (mom_set_kernel_trace) ----
struct TraceHook {
  unsigned long long *buf = nullptr;
  int64_t cap = 0;
  int64_t *count = nullptr;
};
thread_local TraceHook g_trace;
unsigned long long *next_trace_slot(int grid_ctas) {
  // a slot holds kMaxTraceCtas CTAs x 8 stamps: a larger persistent grid is not traced
  if (!g_trace.buf || !g_trace.count || *g_trace.count >= g_trace.cap) return nullptr;
  if (grid_ctas > static_cast<int>(mom::kMaxTraceCtas)) return nullptr;
  return g_trace.buf + (*g_trace.count)++ * (mom::kMaxTraceCtas * 8);
}

// Every launch of the library is also an NVTX range named after its kind (header-only NVTX v3: a few
// ns when no tool is attached), so `ncu --nvtx --nvtx-include "mom.phaseA/"` or nsys can select it.
const char *const kKindNames[] = {"mom.phaseA", "mom.phaseB", "mom.phaseA_f32", "mom.phaseB_f32",
                                  "mom.last_token_gemv", "mom.lm_head", "mom.mlp_fused"};

struct ScopedTiming {
  cudaStream_t s;
  int64_t slot = -1;
  ScopedTiming(cudaStream_t stream, int kind) : s(stream) {
    nvtxRangePushA(kind >= 0 && kind < 7 ? kKindNames[kind] : "mom.launch");
    if (g_hook.ev && g_hook.count && *g_hook.count < g_hook.cap) {
      slot = (*g_hook.count)++;
      g_hook.kinds[slot] = kind;
      cudaEventRecord(g_hook.ev[2 * slot], s);
    }
  }
  ~ScopedTiming() {
    if (slot >= 0) cudaEventRecord(g_hook.ev[2 * slot + 1], s);
    nvtxRangePop();
  }
};

// NVTX range for the copy / collective entries (no timing slot)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

mom_status_t check_pinned(const void *host, const char *who) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, host);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(MOM_ERR_INVALID_ARG, "%s: cannot query host pointer (%s)", who, cudaGetErrorName(e));
  }
  if (at.type != cudaMemoryTypeHost)
    return fail(MOM_ERR_INVALID_ARG, "%s: host buffer is not page-locked (cudaHostAlloc / pin_memory)", who);
  return MOM_OK;
}

// bytes of one mini-sequence's intermediate H_i = min(C, S) * I * w, rounded to 256 B
size_t h_bytes(int64_t S, int64_t I, int64_t C, mom_dtype_t dt) {
  const int64_t rows = C < S ? C : S;
  const size_t b = static_cast<size_t>(rows) * static_cast<size_t>(I) * dtype_bytes(dt);
  return (b + 255) & ~static_cast<size_t>(255);
}

int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// Phase-B tile width: the persistent grid runs ceil(tiles / clusters) waves and a tile's time is
// proportional to its width, so pick the width (multiple of 32, <= 256) minimising
// waves * width -- e.g. hidden 3584: 14 tiles of 256 -> 7 waves, 16 tiles of 224 -> 7 shorter waves.
uint32_t pick_phase_b_width(int64_t rows, int64_t hidden, int cta_group, int num_sms) {
  const int forced = env_int("MOM_NB_B", 0);
  if (forced >= 32 && forced <= 256 && forced % 32 == 0) return static_cast<uint32_t>(forced);
  const int64_t m_tiles = (rows + 128 * cta_group - 1) / (128 * cta_group);
  const int64_t clusters = num_sms / cta_group > 0 ? num_sms / cta_group : 1;
  auto cost = [&](uint32_t nb) { return ((m_tiles * ((hidden + nb - 1) / nb) + clusters - 1) / clusters) * nb; };
  // Narrower tiles cost energy per FLOP (more operand traffic), so only take one that divides
  // hidden exactly and beats 256 by > 5 % in the wave model (measured: +1.2 % at hidden 3584,
  // a loss at hidden 5120 with a partial last tile).
  const int64_t base = cost(256);
  uint32_t best = 256;
  int64_t best_cost = base;
  for (uint32_t nb = 224; nb >= 128; nb -= 32) {
    if (hidden % nb) continue;
    const int64_t c = cost(nb);
    if (c * 100 < base * 95 && c < best_cost) {
      best_cost = c;
      best = nb;
    }
  }
  return best;
}

}  // namespace

extern "C" {

const char *mom_last_error(void) { return g_err; }

mom_status_t mom_set_timing_events(mom_event_t *events, int32_t *kinds, int64_t capacity, int64_t *count) {
  g_err[0] = 0;
  if (!events) {
    g_hook = TimingHook{};
    return MOM_OK;
  }
  if (!kinds || !count || capacity < 1) return fail(MOM_ERR_INVALID_ARG, "mom_set_timing_events: bad arguments");
  g_hook.ev = reinterpret_cast<cudaEvent_t *>(events);
  g_hook.kinds = kinds;
  g_hook.cap = capacity;
  g_hook.count = count;
  return MOM_OK;
}

mom_status_t mom_set_kernel_trace(void *dev_buf, int64_t capacity, int64_t *count) {
  g_err[0] = 0;
  if (!dev_buf) {
    g_trace = TraceHook{};
    return MOM_OK;
  }
  if (!count || capacity < 1 || !aligned16(dev_buf)) return fail(MOM_ERR_INVALID_ARG, "mom_set_kernel_trace: bad arguments");
  g_trace.buf = static_cast<unsigned long long *>(dev_buf);
  g_trace.cap = capacity;
  g_trace.count = count;
  return MOM_OK;
}

const char *mom_version(void) {
  return "libmom 0.4 sm_100a: tcgen05 2-CTA SwiGLU MLP (phase A/B, half-width tail tiles, fused option), fused "
         "all-gather stores, folded RMSNorm (MLP and last token), SIMT f32, PDL GEMVs + argmax, vocab-sharded head, "
         "KV copies, host-input prefetch, NCCL with async-error checks, in-kernel trace, NVTX ranges";
}

int64_t mom_plan_minseq(int64_t S, int64_t C, int64_t *starts, int64_t *lens, int64_t cap) {
  if (S < 1 || C < 1) return -1;
  const int64_t M = (S + C - 1) / C;  // Alg. 1: M = ceil(S/C)
  for (int64_t i = 0; i < M && i < cap; ++i) {
    const int64_t r0 = i * C;
    const int64_t r1 = (r0 + C < S) ? r0 + C : S;
    if (starts) starts[i] = r0;
    if (lens) lens[i] = r1 - r0;
  }
  return M;
}

size_t mom_mlp_minseq_workspace_bytes(int64_t S, int64_t hidden, int64_t intermediate, int64_t C,
                                      mom_dtype_t dt) {
  (void)hidden;
  if (S < 1 || intermediate < 1 || C < 1 || !valid_dtype(dt)) return 0;
  const size_t h = h_bytes(S, intermediate, C, dt);  // one mini-sequence's H_i: C * I elements (Eq. 3)
  if (dt == MOM_F32) return h;
  const int64_t rows = C < S ? C : S;  // + the fused kernel's per-row-block counters (<= ~4 KB at C = 8192)
  return h + ((mom::mlp_tc_ready_counters(static_cast<uint32_t>(rows)) * 4 + 255) & ~static_cast<size_t>(255));
}

}  // extern "C"

namespace {

mom_status_t validate_minseq(const char *who, const void *x, const void *residual, const void *w_gate,
                             const void *w_up, const void *w_down, const void *out, int64_t S, int64_t hidden,
                             int64_t intermediate, int64_t C, mom_dtype_t dt, const void *workspace,
                             size_t workspace_bytes) {
  if (!x || !w_gate || !w_up || !w_down || !out || !workspace) return fail(MOM_ERR_INVALID_ARG, "%s: null pointer", who);
  if (S < 1 || hidden < 1 || intermediate < 1 || C < 1)
    return fail(MOM_ERR_INVALID_ARG, "%s: S, hidden, intermediate, minseq_len must be >= 1", who);
  if (!valid_dtype(dt)) return fail(MOM_ERR_INVALID_ARG, "%s: bad dtype %d", who, (int)dt);
  const size_t w = dtype_bytes(dt);
  if ((hidden * w) % 16 || (intermediate * w) % 16)
    return fail(MOM_ERR_INVALID_ARG, "%s: row pitch must be a multiple of 16 bytes", who);
  if (!aligned16(x) || !aligned16(residual) || !aligned16(w_gate) || !aligned16(w_up) || !aligned16(w_down) ||
      !aligned16(out) || !aligned16(workspace))
    return fail(MOM_ERR_INVALID_ARG, "%s: pointers must be 16-byte aligned", who);
  if (S > INT32_MAX || hidden > INT32_MAX || intermediate > INT32_MAX)
    return fail(MOM_ERR_INVALID_ARG, "%s: dimension exceeds int32", who);
  const size_t act_bytes = static_cast<size_t>(S) * hidden * w;
  if (partial_overlap(out, act_bytes, x, act_bytes) || partial_overlap(out, act_bytes, residual, act_bytes))
    return fail(MOM_ERR_INVALID_ARG, "%s: out partially overlaps x or residual", who);
  const size_t need = mom_mlp_minseq_workspace_bytes(S, hidden, intermediate, C, dt);
  if (workspace_bytes < need)
    return fail(MOM_ERR_WORKSPACE, "%s: workspace %zu < required %zu bytes", who, workspace_bytes, need);
  return MOM_OK;
}

// Alg. 1 P:109-113.  When x_host is non-null, mini-sequence i's rows are first copied host->device
// (x_host -> x) on `copy`, and `stream` waits for exactly those rows before running MLP(A_i): the
// transfer of A_{i+1} overlaps the tensor-core work on A_i.
mom_status_t run_minseq(const void *x, const void *residual, const void *w_gate, const void *w_up,
                        const void *w_down, void *out, int64_t S, int64_t hidden, int64_t intermediate, int64_t C,
                        mom_dtype_t dt, void *workspace, cudaStream_t stream, const void *x_host,
                        cudaStream_t copy, const float *norm_eps = nullptr, void *const *peers = nullptr,
                        int n_peers = 0) {
  int num_sms = 0;
  if (num_sms_current(&num_sms) != 0) return fail(MOM_ERR_CUDA, "mom_mlp_minseq_fwd: no CUDA device");
  const int64_t M = (S + C - 1) / C;  // Alg. 1
  const size_t w = dtype_bytes(dt);
  const int cta_group = env_int("MOM_CTA_GROUP", 2) == 1 ? 1 : 2;
  const uint32_t group_a = static_cast<uint32_t>(env_int("MOM_GROUP_M_A", 0));
  const uint32_t group_b = static_cast<uint32_t>(env_int("MOM_GROUP_M_B", 0));
  const uint32_t policy = static_cast<uint32_t>(env_int("MOM_TMA_POLICY", 0));
  // Two launches per mini-sequence by default: the fused single launch removes the inter-phase
  // tail but runs phase-A and phase-B tiles concurrently, which costs more DRAM traffic, and on
  // the power-capped B200 that energy costs more clock than the tail (energy sweep, round 1).
  const bool fused = env_int("MOM_FUSED", 0) != 0;
  const bool mlp_pdl = env_int("MOM_MLP_PDL", 1) != 0;
  // phase-A wave tail as half-width tiles (bitwise neutral: same K order per output element)
  const bool half_tail = env_int("MOM_HALF_TAIL", 1) != 0;
  CUtensorMap tm_wg, tm_wu, tm_wd, tm_wg_h, tm_wu_h;
  mom_status_t st;
  if (dt == MOM_BF16) {
    if ((st = make_tmap(&tm_wg, w_gate, intermediate, hidden, "w_gate")) != MOM_OK) return st;
    if ((st = make_tmap(&tm_wu, w_up, intermediate, hidden, "w_up")) != MOM_OK) return st;
    if (half_tail) {
      if ((st = make_tmap(&tm_wg_h, w_gate, intermediate, hidden, "w_gate", 64)) != MOM_OK) return st;
      if ((st = make_tmap(&tm_wu_h, w_up, intermediate, hidden, "w_up", 64)) != MOM_OK) return st;
    }
  }
  uint32_t wd_box = 0;  // W_down map is (re)encoded when the phase-B tile width changes
  for (int64_t i = 0; i < M; ++i) {  // Alg. 1: for i = 1..M (sequential on `stream`)
    const int64_t r0 = i * C;
    const int64_t rows = (r0 + C < S) ? C : S - r0;
    const size_t off = static_cast<size_t>(r0) * hidden * w;  // byte offset of A_i / O_i
    cudaError_t e;
    if (x_host) {
      e = cudaMemcpyAsync(const_cast<char *>(static_cast<const char *>(x)) + off,
                          static_cast<const char *>(x_host) + off, static_cast<size_t>(rows) * hidden * w,
                          cudaMemcpyHostToDevice, copy);
      if (e != cudaSuccess) return cuda_fail(e, "mini-sequence H2D");
      cudaEvent_t landed;
      if ((e = cudaEventCreateWithFlags(&landed, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "event create");
      e = cudaEventRecord(landed, copy);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, landed, 0);
      cudaEventDestroy(landed);
      if (e != cudaSuccess) return cuda_fail(e, "mini-sequence H2D ordering");
    }
    const void *xi = static_cast<const char *>(x) + off;
    const void *ri = residual ? static_cast<const char *>(residual) + off : nullptr;
    void *oi = static_cast<char *>(out) + off;  // concat: O_i lands at its rows
    if (dt == MOM_F32) {
      float *h = static_cast<float *>(workspace);
      {
        ScopedTiming tm(stream, 2);
        e = mom::launch_phase_a_f32(static_cast<const float *>(xi), static_cast<const float *>(w_gate),
                                    static_cast<const float *>(w_up), h, (int)rows, (int)hidden, (int)intermediate,
                                    stream);
      }
      if (e != cudaSuccess) return cuda_fail(e, "phase A (f32)");
      {
        ScopedTiming tm(stream, 3);
        e = mom::launch_phase_b_f32(h, static_cast<const float *>(w_down), static_cast<const float *>(ri),
                                    static_cast<float *>(oi), (int)rows, (int)hidden, (int)intermediate, stream);
      }
      if (e != cudaSuccess) return cuda_fail(e, "phase B (f32)");
      continue;
    }
    __nv_bfloat16 *h = static_cast<__nv_bfloat16 *>(workspace);
    // Per-mini-sequence maps: the row bound is C_i, so TMA zero-fills loads past the end of
    // this mini-sequence and no tile reads another mini-sequence's rows.
    CUtensorMap tm_x, tm_h;
    if ((st = make_tmap(&tm_x, xi, rows, hidden, "x_i")) != MOM_OK) return st;
    if ((st = make_tmap(&tm_h, h, rows, intermediate, "h_i")) != MOM_OK) return st;
    mom::TcMlpArgs a{};
    a.tm_x = &tm_x; a.tm_wg = &tm_wg; a.tm_wu = &tm_wu; a.tm_h = &tm_h; a.tm_wd = &tm_wd;
    a.tm_wg_h = half_tail ? &tm_wg_h : nullptr;
    a.tm_wu_h = half_tail ? &tm_wu_h : nullptr;
    a.rows = (uint32_t)rows; a.d = (uint32_t)hidden; a.I = (uint32_t)intermediate;
    a.h = h; a.out = static_cast<__nv_bfloat16 *>(oi); a.residual = static_cast<const __nv_bfloat16 *>(ri);
    a.cta_group = cta_group; a.policy = policy; a.num_sms = num_sms;
    a.nb = pick_phase_b_width(rows, hidden, cta_group, num_sms);
    if (a.nb != wd_box) {  // B halves of phase B are nb/2 rows of W_down per CTA
      if ((st = make_tmap(&tm_wd, w_down, hidden, intermediate, "w_down", a.nb / 2)) != MOM_OK) return st;
      wd_box = a.nb;
    }
    a.coalesced_a = static_cast<uint32_t>(env_int("MOM_EPI_A_COALESCED", 1));
    a.fast_silu = static_cast<uint32_t>(env_int("MOM_FAST_SILU", 1));
    a.epi_hint = static_cast<uint32_t>(env_int("MOM_EPI_L2_HINT", 0));
    a.ready = reinterpret_cast<uint32_t *>(static_cast<char *>(workspace) + h_bytes(S, intermediate, C, dt));
    // f1: every O_i row must reach every peer.  Rows of mini-sequence i-1 (final once its phase B
    // completed) are forwarded by warps 2-3 of this mini-sequence's phase-A launch, so the NVLink
    // traffic overlaps the tensor-core work; only the last mini-sequence's rows are stored to
    // the peers by the phase-B epilogue that produces them.
    const bool fwd_mode = env_int("MOM_GATHER_FORWARD", 1) != 0;
    a.n_peers = (!fwd_mode || i == M - 1) ? static_cast<uint32_t>(n_peers) : 0u;
    for (int k = 0; k < n_peers; ++k) a.peer_out[k] = reinterpret_cast<__nv_bfloat16 *>(static_cast<char *>(peers[k]) + off);
    a.fwd_src = nullptr;
    a.fwd_rows = 0;
    a.n_fwd = 0;
    if (fwd_mode && n_peers > 0 && i > 0) {
      const size_t prev = static_cast<size_t>(r0 - C) * hidden * w;
      a.fwd_src = reinterpret_cast<const __nv_bfloat16 *>(static_cast<const char *>(out) + prev);
      a.fwd_rows = static_cast<uint32_t>(C);
      a.n_fwd = static_cast<uint32_t>(n_peers);
      for (int k = 0; k < n_peers; ++k) a.fwd_dst[k] = reinterpret_cast<__nv_bfloat16 *>(static_cast<char *>(peers[k]) + prev);
    }
    if (norm_eps) {
      // folded RMSNorm (f3): 1/rms of this mini-sequence's rows, after H_i and the counters
      float *inv = reinterpret_cast<float *>(static_cast<char *>(workspace) +
                                             mom_mlp_minseq_workspace_bytes(S, hidden, intermediate, C, dt));
      e = mom::launch_row_inv_rms(static_cast<const __nv_bfloat16 *>(xi), inv, (int)rows, (int)hidden, *norm_eps,
                                  num_sms, stream);
      if (e != cudaSuccess) return cuda_fail(e, "row 1/rms");
      a.row_scale = inv;
    }
    if (fused) {
      // one persistent launch: H_i = Swish(A_i Wg^T) (.) A_i Wu^T and O_i = R_i + H_i Wd^T,
      // O_i written at rows r0..; phase-B tiles wait on per-row-block counters
      e = cudaMemsetAsync(a.ready, 0, mom::mlp_tc_ready_counters((uint32_t)rows) * sizeof(uint32_t), stream);
      if (e != cudaSuccess) return cuda_fail(e, "counter reset");
      a.group_m = group_a;
      ScopedTiming tm(stream, 6);
      a.trace = next_trace_slot(num_sms);
      e = mom::launch_mlp_tc(a, 2, stream);
      if (e != cudaSuccess) return cuda_fail(e, "fused MLP (tcgen05)");
      continue;
    }
    a.group_m = group_a;
    // PDL: phase A of mini-sequence i > 0 may start on the SMs the previous phase B frees and
    // stream X_i / weights while that phase B finishes (its epilogue waits before storing H_i);
    // phase B may start its prologue under phase A's tail.  Not after a host->device wait.
    a.pdl = mlp_pdl && i > 0 && !x_host;
    {
      ScopedTiming tm(stream, 0);
      a.trace = next_trace_slot(num_sms);
      e = mom::launch_mlp_tc(a, 0, stream);  // H_i = Swish(A_i Wg^T) (.) A_i Wu^T
    }
    if (e != cudaSuccess) return cuda_fail(e, "phase A (tcgen05)");
    a.group_m = group_b;
    a.group_n = static_cast<uint32_t>(env_int("MOM_RASTER_B_COLS", 0));
    a.fwd_src = nullptr;  // forwarding rides on the phase-A launch only
    a.n_fwd = 0;
    a.pdl = mlp_pdl;
    {
      ScopedTiming tm(stream, 1);
      a.trace = next_trace_slot(num_sms);
      e = mom::launch_mlp_tc(a, 1, stream);  // O_i = R_i + H_i Wd^T, written at rows r0..
    }
    if (e != cudaSuccess) return cuda_fail(e, "phase B (tcgen05)");
  }
  return MOM_OK;
}

}  // namespace

extern "C" {

mom_status_t mom_mlp_minseq_fwd(const void *x, const void *residual, const void *w_gate, const void *w_up,
                                const void *w_down, void *out, int64_t S, int64_t hidden, int64_t intermediate,
                                int64_t C, mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                                mom_stream_t stream) {
  g_err[0] = 0;
  mom_status_t st = validate_minseq("mom_mlp_minseq_fwd", x, residual, w_gate, w_up, w_down, out, S, hidden,
                                    intermediate, C, dt, workspace, workspace_bytes);
  if (st != MOM_OK) return st;
  return run_minseq(x, residual, w_gate, w_up, w_down, out, S, hidden, intermediate, C, dt, workspace,
                    static_cast<cudaStream_t>(stream), nullptr, nullptr);
}

mom_status_t mom_mlp_minseq_fwd_gather(const void *x, const void *residual, const void *w_gate, const void *w_up,
                                       const void *w_down, void *out, void *const *peer_out, int n_peers, int64_t S,
                                       int64_t hidden, int64_t intermediate, int64_t C, mom_dtype_t dt,
                                       void *workspace, size_t workspace_bytes, mom_stream_t stream) {
  g_err[0] = 0;
  mom_status_t st = validate_minseq("mom_mlp_minseq_fwd_gather", x, residual, w_gate, w_up, w_down, out, S, hidden,
                                    intermediate, C, dt, workspace, workspace_bytes);
  if (st != MOM_OK) return st;
  if (n_peers < 0 || n_peers > static_cast<int>(mom::kMaxPeers) || (n_peers > 0 && !peer_out))
    return fail(MOM_ERR_INVALID_ARG, "mom_mlp_minseq_fwd_gather: 0 <= n_peers <= %u", mom::kMaxPeers);
  for (int k = 0; k < n_peers; ++k)
    if (!peer_out[k] || !aligned16(peer_out[k]))
      return fail(MOM_ERR_INVALID_ARG, "mom_mlp_minseq_fwd_gather: peer %d pointer null or misaligned", k);
  if (dt != MOM_BF16 && n_peers > 0)
    return fail(MOM_ERR_UNSUPPORTED, "mom_mlp_minseq_fwd_gather: peer stores are bf16 (tcgen05 path) only");
  return run_minseq(x, residual, w_gate, w_up, w_down, out, S, hidden, intermediate, C, dt, workspace,
                    static_cast<cudaStream_t>(stream), nullptr, nullptr, nullptr, peer_out, n_peers);
}

mom_status_t mom_ipc_get_handle(const void *dev_ptr, void *handle_out, int64_t *offset_out) {
  g_err[0] = 0;
  if (!dev_ptr || !handle_out || !offset_out) return fail(MOM_ERR_INVALID_ARG, "mom_ipc_get_handle: null pointer");
  // the IPC handle names the whole allocation: find its base (torch sub-allocates)
  using RangeFn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
  static RangeFn range = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<RangeFn>(p)
               : nullptr;
  }();
  if (!range) return fail(MOM_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(MOM_ERR_INVALID_ARG, "mom_ipc_get_handle: not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
  if (e != cudaSuccess)
    return cuda_fail(e, "cudaIpcGetMemHandle (the allocation is not IPC-exportable -- e.g. torch's "
                        "expandable_segments / cuMemCreate memory; use the NCCL all-gather path)");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return MOM_OK;
}

mom_status_t mom_ipc_open_handle(const void *handle, int64_t offset, void **dev_ptr_out) {
  g_err[0] = 0;
  if (!handle || !dev_ptr_out || offset < 0) return fail(MOM_ERR_INVALID_ARG, "mom_ipc_open_handle: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void *base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  *dev_ptr_out = static_cast<char *>(base) + offset;
  return MOM_OK;
}

mom_status_t mom_ipc_close(void *dev_ptr, int64_t offset) {
  g_err[0] = 0;
  if (!dev_ptr) return fail(MOM_ERR_INVALID_ARG, "mom_ipc_close: null pointer");
  cudaError_t e = cudaIpcCloseMemHandle(static_cast<char *>(dev_ptr) - offset);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return MOM_OK;
}

}  // extern "C"

namespace {
mom_status_t from_host_impl(const char *who, const void *x_host_pinned, void *x, const void *residual,
                            const void *w_gate, const void *w_up, const void *w_down, void *out,
                            void *const *peer_out, int n_peers, int64_t S, int64_t hidden, int64_t intermediate,
                            int64_t C, mom_dtype_t dt, void *workspace, size_t workspace_bytes, mom_stream_t stream,
                            mom_stream_t copy_stream, mom_event_t x_free) {
  g_err[0] = 0;
  if (!x_host_pinned) return fail(MOM_ERR_INVALID_ARG, "%s: null host pointer", who);
  mom_status_t st = validate_minseq(who, x, residual, w_gate, w_up, w_down, out, S, hidden, intermediate, C, dt,
                                    workspace, workspace_bytes);
  if (st != MOM_OK) return st;
  if (n_peers < 0 || n_peers > static_cast<int>(mom::kMaxPeers) || (n_peers > 0 && !peer_out))
    return fail(MOM_ERR_INVALID_ARG, "%s: 0 <= n_peers <= %u", who, mom::kMaxPeers);
  for (int k = 0; k < n_peers; ++k)
    if (!peer_out[k] || !aligned16(peer_out[k]))
      return fail(MOM_ERR_INVALID_ARG, "%s: peer %d pointer null or misaligned", who, k);
  if (dt != MOM_BF16 && n_peers > 0) return fail(MOM_ERR_UNSUPPORTED, "%s: peer stores are bf16 only", who);
  if ((st = check_pinned(x_host_pinned, who)) != MOM_OK) return st;
  if (copy_stream == stream) return fail(MOM_ERR_INVALID_ARG, "%s: copy_stream must differ from stream", who);
  cudaStream_t s = static_cast<cudaStream_t>(stream), cp = static_cast<cudaStream_t>(copy_stream);
  cudaError_t e;
  if (x_free) {
    // the caller names the point after which x is free (double-buffered inputs: prefetch)
    e = cudaStreamWaitEvent(cp, static_cast<cudaEvent_t>(x_free), 0);
    if (e != cudaSuccess) return cuda_fail(e, "x_free ordering");
  } else {
    // the copy stream must not start writing x before earlier work on `stream` is done with it
    cudaEvent_t ready;
    e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "event create");
    e = cudaEventRecord(ready, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cp, ready, 0);
    cudaEventDestroy(ready);
    if (e != cudaSuccess) return cuda_fail(e, "stream ordering");
  }
  return run_minseq(x, residual, w_gate, w_up, w_down, out, S, hidden, intermediate, C, dt, workspace, s,
                    x_host_pinned, cp, nullptr, peer_out, n_peers);
}
}  // namespace

extern "C" {

mom_status_t mom_mlp_minseq_fwd_from_host(const void *x_host_pinned, void *x, const void *residual,
                                          const void *w_gate, const void *w_up, const void *w_down, void *out,
                                          int64_t S, int64_t hidden, int64_t intermediate, int64_t C,
                                          mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                                          mom_stream_t stream, mom_stream_t copy_stream, mom_event_t x_free) {
  return from_host_impl("mom_mlp_minseq_fwd_from_host", x_host_pinned, x, residual, w_gate, w_up, w_down, out,
                        nullptr, 0, S, hidden, intermediate, C, dt, workspace, workspace_bytes, stream, copy_stream,
                        x_free);
}

mom_status_t mom_mlp_minseq_fwd_from_host_gather(const void *x_host_pinned, void *x, const void *residual,
                                                 const void *w_gate, const void *w_up, const void *w_down,
                                                 void *out, void *const *peer_out, int n_peers, int64_t S,
                                                 int64_t hidden, int64_t intermediate, int64_t C, mom_dtype_t dt,
                                                 void *workspace, size_t workspace_bytes, mom_stream_t stream,
                                                 mom_stream_t copy_stream, mom_event_t x_free) {
  return from_host_impl("mom_mlp_minseq_fwd_from_host_gather", x_host_pinned, x, residual, w_gate, w_up, w_down,
                        out, peer_out, n_peers, S, hidden, intermediate, C, dt, workspace, workspace_bytes, stream,
                        copy_stream, x_free);
}

mom_status_t mom_fold_norm_gain(const void *w, const void *norm_gain, void *w_folded, int64_t rows, int64_t cols,
                                mom_dtype_t dt, mom_stream_t stream) {
  g_err[0] = 0;
  if (!w || !norm_gain || !w_folded) return fail(MOM_ERR_INVALID_ARG, "mom_fold_norm_gain: null pointer");
  if (rows < 1 || cols < 1) return fail(MOM_ERR_INVALID_ARG, "mom_fold_norm_gain: sizes must be >= 1");
  if (dt != MOM_BF16) return fail(MOM_ERR_UNSUPPORTED, "mom_fold_norm_gain: bf16 only");
  if (cols % 8 || !aligned16(w) || !aligned16(norm_gain) || !aligned16(w_folded))
    return fail(MOM_ERR_INVALID_ARG, "mom_fold_norm_gain: 16-byte alignment and cols %% 8 == 0 required");
  if (partial_overlap(w, rows * cols * 2, w_folded, rows * cols * 2))
    return fail(MOM_ERR_INVALID_ARG, "mom_fold_norm_gain: w_folded partially overlaps w");
  int num_sms = 0;
  if (num_sms_current(&num_sms) != 0) return fail(MOM_ERR_CUDA, "mom_fold_norm_gain: no CUDA device");
  cudaError_t e = mom::launch_fold_gain(static_cast<const __nv_bfloat16 *>(w),
                                        static_cast<const __nv_bfloat16 *>(norm_gain),
                                        static_cast<__nv_bfloat16 *>(w_folded), rows, cols, num_sms,
                                        static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fold gain");
  return MOM_OK;
}

size_t mom_mlp_minseq_rmsnorm_workspace_bytes(int64_t S, int64_t hidden, int64_t intermediate, int64_t C,
                                              mom_dtype_t dt) {
  const size_t h = mom_mlp_minseq_workspace_bytes(S, hidden, intermediate, C, dt);
  if (h == 0) return 0;
  const int64_t rows = C < S ? C : S;
  return h + ((static_cast<size_t>(rows) * 4 + 255) & ~static_cast<size_t>(255));
}

mom_status_t mom_mlp_minseq_rmsnorm_fwd(const void *x, const void *w_gate_folded, const void *w_up_folded,
                                        const void *w_down, void *out, int64_t S, int64_t hidden,
                                        int64_t intermediate, int64_t C, float eps, mom_dtype_t dt,
                                        void *workspace, size_t workspace_bytes, mom_stream_t stream) {
  g_err[0] = 0;
  if (dt != MOM_BF16) return fail(MOM_ERR_UNSUPPORTED, "mom_mlp_minseq_rmsnorm_fwd: bf16 only");
  if (!(eps >= 0.0f)) return fail(MOM_ERR_INVALID_ARG, "mom_mlp_minseq_rmsnorm_fwd: eps must be >= 0");
  mom_status_t st = validate_minseq("mom_mlp_minseq_rmsnorm_fwd", x, x, w_gate_folded, w_up_folded, w_down, out, S,
                                    hidden, intermediate, C, dt, workspace, workspace_bytes);
  if (st != MOM_OK) return st;
  const size_t need = mom_mlp_minseq_rmsnorm_workspace_bytes(S, hidden, intermediate, C, dt);
  if (workspace_bytes < need)
    return fail(MOM_ERR_WORKSPACE, "mom_mlp_minseq_rmsnorm_fwd: workspace %zu < required %zu bytes", workspace_bytes,
                need);
  return run_minseq(x, x, w_gate_folded, w_up_folded, w_down, out, S, hidden, intermediate, C, dt, workspace,
                    static_cast<cudaStream_t>(stream), nullptr, nullptr, &eps);
}

size_t mom_mlp_last_token_workspace_bytes(int64_t intermediate) {
  if (intermediate < 1) return 0;
  return ((static_cast<size_t>(intermediate) * 4) + 255) & ~static_cast<size_t>(255);  // h, fp32
}

static mom_status_t last_token_impl(const void *x_last, const void *residual_last, const void *w_gate,
                                    const void *w_up, const void *w_down, void *out_last, int64_t hidden,
                                    int64_t intermediate, mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                                    mom_stream_t stream, float norm_eps) {
  g_err[0] = 0;
  if (!x_last || !w_gate || !w_up || !w_down || !out_last || !workspace)
    return fail(MOM_ERR_INVALID_ARG, "mom_mlp_last_token: null pointer");
  if (hidden < 1 || intermediate < 1) return fail(MOM_ERR_INVALID_ARG, "mom_mlp_last_token: sizes must be >= 1");
  if (!valid_dtype(dt)) return fail(MOM_ERR_INVALID_ARG, "mom_mlp_last_token: bad dtype");
  const size_t w = dtype_bytes(dt);
  if ((hidden * w) % 16 || (intermediate * w) % 16)
    return fail(MOM_ERR_INVALID_ARG, "mom_mlp_last_token: row pitch must be a multiple of 16 bytes");
  if (!aligned16(x_last) || !aligned16(residual_last) || !aligned16(w_gate) || !aligned16(w_up) ||
      !aligned16(w_down) || !aligned16(out_last) || !aligned16(workspace))
    return fail(MOM_ERR_INVALID_ARG, "mom_mlp_last_token: pointers must be 16-byte aligned");
  if (partial_overlap(out_last, hidden * w, x_last, hidden * w) ||
      partial_overlap(out_last, hidden * w, residual_last, hidden * w))
    return fail(MOM_ERR_INVALID_ARG, "mom_mlp_last_token: out_last partially overlaps an input");
  if (x_last == out_last && residual_last != out_last)
    return fail(MOM_ERR_INVALID_ARG, "mom_mlp_last_token: out_last may alias x_last only when residual_last does too");
  if (hidden > (1 << 24) || intermediate > (1 << 24))
    return fail(MOM_ERR_UNSUPPORTED, "mom_mlp_last_token: staging buffers limit hidden/intermediate to 2^24");
  const size_t need = mom_mlp_last_token_workspace_bytes(intermediate);
  if (workspace_bytes < need) return fail(MOM_ERR_WORKSPACE, "mom_mlp_last_token: workspace %zu < %zu", workspace_bytes, need);
  if (static_cast<size_t>(intermediate) * 4 > 227 * 1024 || static_cast<size_t>(hidden) * 4 > 227 * 1024)
    return fail(MOM_ERR_UNSUPPORTED, "mom_mlp_last_token: vector does not fit in shared memory");
  int num_sms = 0;
  if (num_sms_current(&num_sms) != 0) return fail(MOM_ERR_CUDA, "mom_mlp_last_token: no CUDA device");
  cudaError_t e;
  ScopedTiming tm(static_cast<cudaStream_t>(stream), 4);
  e = mom::launch_last_token_mlp(x_last, residual_last, w_gate, w_up, w_down, out_last,
                                             static_cast<float *>(workspace), (int)hidden, (int)intermediate,
                                             dt == MOM_BF16, num_sms, static_cast<cudaStream_t>(stream), norm_eps);
  if (e != cudaSuccess) return cuda_fail(e, "last-token MLP");
  return MOM_OK;
}

mom_status_t mom_mlp_last_token(const void *x_last, const void *residual_last, const void *w_gate,
                                const void *w_up, const void *w_down, void *out_last, int64_t hidden,
                                int64_t intermediate, mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                                mom_stream_t stream) {
  return last_token_impl(x_last, residual_last, w_gate, w_up, w_down, out_last, hidden, intermediate, dt, workspace,
                         workspace_bytes, stream, -1.0f);
}

mom_status_t mom_mlp_last_token_rmsnorm(const void *x_last, const void *w_gate_folded, const void *w_up_folded,
                                        const void *w_down, void *out_last, int64_t hidden, int64_t intermediate,
                                        float eps, mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                                        mom_stream_t stream) {
  g_err[0] = 0;
  if (!(eps >= 0.0f)) return fail(MOM_ERR_INVALID_ARG, "mom_mlp_last_token_rmsnorm: eps must be >= 0");
  return last_token_impl(x_last, x_last, w_gate_folded, w_up_folded, w_down, out_last, hidden, intermediate, dt,
                         workspace, workspace_bytes, stream, eps);
}

size_t mom_lm_head_workspace_bytes(int64_t vocab) {
  if (vocab < 1) return 0;
  return 256 * 4 * sizeof(unsigned long long);  // per-block partial maxima (<= 4 per SM, <= 256 SMs)
}

mom_status_t mom_lm_head_last(const void *h_last, const void *norm_gain, float eps, const void *w_head,
                              float *logits, int32_t *argmax, int64_t hidden, int64_t vocab, mom_dtype_t dt,
                              void *workspace, size_t workspace_bytes, mom_stream_t stream) {
  g_err[0] = 0;
  if (!h_last || !w_head || !argmax || !workspace) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_last: null pointer");
  if (hidden < 1 || vocab < 1) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_last: sizes must be >= 1");
  if (!valid_dtype(dt)) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_last: bad dtype");
  if (norm_gain && !(eps >= 0.0f)) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_last: eps must be >= 0");
  const size_t w = dtype_bytes(dt);
  if ((hidden * w) % 16) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_last: row pitch must be a multiple of 16 bytes");
  if (!aligned16(h_last) || !aligned16(norm_gain) || !aligned16(w_head) || !aligned16(logits) ||
      !aligned16(workspace) || (reinterpret_cast<uintptr_t>(argmax) & 3))
    return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_last: misaligned pointer");
  if (vocab > INT32_MAX - 1) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_last: vocab exceeds int32");
  if (static_cast<size_t>(hidden) * 4 > 200 * 1024)
    return fail(MOM_ERR_UNSUPPORTED, "mom_lm_head_last: hidden too large for shared-memory staging");
  const size_t need = mom_lm_head_workspace_bytes(vocab);
  if (workspace_bytes < need) return fail(MOM_ERR_WORKSPACE, "mom_lm_head_last: workspace %zu < %zu", workspace_bytes, need);
  int num_sms = 0;
  if (num_sms_current(&num_sms) != 0) return fail(MOM_ERR_CUDA, "mom_lm_head_last: no CUDA device");
  if (num_sms > 256) num_sms = 256;
  cudaError_t e;
  ScopedTiming tm(static_cast<cudaStream_t>(stream), 5);
  e = mom::launch_lm_head(h_last, norm_gain, eps, w_head, logits, argmax, nullptr, 0,
                                      static_cast<unsigned long long *>(workspace), (int)hidden, (int)vocab,
                                      dt == MOM_BF16, num_sms, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "lm head");
  return MOM_OK;
}

mom_status_t mom_lm_head_shard(const void *h_last, const void *norm_gain, float eps, const void *w_head_shard,
                               int64_t vocab_offset, int64_t vocab_shard, float *logits_shard, uint64_t *best_key,
                               int64_t hidden, mom_dtype_t dt, void *workspace, size_t workspace_bytes,
                               mom_stream_t stream) {
  g_err[0] = 0;
  if (!h_last || !w_head_shard || !best_key || !workspace)
    return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_shard: null pointer");
  if (hidden < 1 || vocab_shard < 1 || vocab_offset < 0)
    return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_shard: bad sizes");
  if (!valid_dtype(dt)) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_shard: bad dtype");
  if (norm_gain && !(eps >= 0.0f)) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_shard: eps must be >= 0");
  const size_t w = dtype_bytes(dt);
  if ((hidden * w) % 16) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_shard: row pitch must be a multiple of 16 bytes");
  if (!aligned16(h_last) || !aligned16(norm_gain) || !aligned16(w_head_shard) || !aligned16(logits_shard) ||
      !aligned16(workspace) || (reinterpret_cast<uintptr_t>(best_key) & 7))
    return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_shard: misaligned pointer");
  if (vocab_offset + vocab_shard > INT32_MAX - 1) return fail(MOM_ERR_INVALID_ARG, "mom_lm_head_shard: vocab exceeds int32");
  if (static_cast<size_t>(hidden) * 4 > 200 * 1024)
    return fail(MOM_ERR_UNSUPPORTED, "mom_lm_head_shard: hidden too large for shared-memory staging");
  const size_t need = mom_lm_head_workspace_bytes(vocab_shard);
  if (workspace_bytes < need) return fail(MOM_ERR_WORKSPACE, "mom_lm_head_shard: workspace %zu < %zu", workspace_bytes, need);
  int num_sms = 0;
  if (num_sms_current(&num_sms) != 0) return fail(MOM_ERR_CUDA, "mom_lm_head_shard: no CUDA device");
  if (num_sms > 256) num_sms = 256;
  ScopedTiming tm(static_cast<cudaStream_t>(stream), 5);
  cudaError_t e = mom::launch_lm_head(h_last, norm_gain, eps, w_head_shard, logits_shard, nullptr,
                                      reinterpret_cast<unsigned long long *>(best_key), (int)vocab_offset,
                                      static_cast<unsigned long long *>(workspace), (int)hidden, (int)vocab_shard,
                                      dt == MOM_BF16, num_sms, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "lm head shard");
  return MOM_OK;
}

mom_status_t mom_kv_offload(const void *kv_dev, void *kv_host_pinned, size_t bytes, mom_stream_t producer_stream,
                            mom_stream_t copy_stream, mom_event_t done) {
  g_err[0] = 0;
  if (!kv_dev || !kv_host_pinned || bytes < 1) return fail(MOM_ERR_INVALID_ARG, "mom_kv_offload: null pointer or zero bytes");
  if (!aligned16(kv_dev)) return fail(MOM_ERR_INVALID_ARG, "mom_kv_offload: kv_dev must be 16-byte aligned");
  mom_status_t st = check_pinned(kv_host_pinned, "mom_kv_offload");
  if (st != MOM_OK) return st;
  cudaStream_t prod = static_cast<cudaStream_t>(producer_stream), cp = static_cast<cudaStream_t>(copy_stream);
  if (prod != cp) {
    cudaEvent_t ready;
    cudaError_t e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "mom_kv_offload: event create");
    e = cudaEventRecord(ready, prod);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cp, ready, 0);
    cudaEventDestroy(ready);  // released once the recorded work completes
    if (e != cudaSuccess) return cuda_fail(e, "mom_kv_offload: stream ordering");
  }
  NvtxRange nvtx("mom.kv_offload");
  cudaError_t e = cudaMemcpyAsync(kv_host_pinned, kv_dev, bytes, cudaMemcpyDeviceToHost, cp);
  if (e != cudaSuccess) return cuda_fail(e, "mom_kv_offload: cudaMemcpyAsync D2H");
  if (done) {
    e = cudaEventRecord(static_cast<cudaEvent_t>(done), cp);
    if (e != cudaSuccess) return cuda_fail(e, "mom_kv_offload: event record");
  }
  return MOM_OK;
}

mom_status_t mom_kv_reload(const void *kv_host_pinned, void *kv_dev, size_t bytes, mom_stream_t copy_stream,
                           mom_event_t done) {
  g_err[0] = 0;
  if (!kv_dev || !kv_host_pinned || bytes < 1) return fail(MOM_ERR_INVALID_ARG, "mom_kv_reload: null pointer or zero bytes");
  if (!aligned16(kv_dev)) return fail(MOM_ERR_INVALID_ARG, "mom_kv_reload: kv_dev must be 16-byte aligned");
  mom_status_t st = check_pinned(kv_host_pinned, "mom_kv_reload");
  if (st != MOM_OK) return st;
  cudaStream_t cp = static_cast<cudaStream_t>(copy_stream);
  NvtxRange nvtx("mom.kv_reload");
  cudaError_t e = cudaMemcpyAsync(kv_dev, kv_host_pinned, bytes, cudaMemcpyHostToDevice, cp);
  if (e != cudaSuccess) return cuda_fail(e, "mom_kv_reload: cudaMemcpyAsync H2D");
  if (done) {
    e = cudaEventRecord(static_cast<cudaEvent_t>(done), cp);
    if (e != cudaSuccess) return cuda_fail(e, "mom_kv_reload: event record");
  }
  return MOM_OK;
}

// ------------------------------------------------------------------------ NCCL (dlopen)
namespace {
typedef struct { char internal[128]; } nccl_uid_t;
typedef int (*nccl_get_uid_fn)(nccl_uid_t *);
typedef int (*nccl_init_fn)(void **, int, nccl_uid_t, int);
typedef int (*nccl_destroy_fn)(void *);
typedef int (*nccl_allgather_fn)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*nccl_allreduce_fn)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef const char *(*nccl_errstr_fn)(int);
typedef int (*nccl_async_err_fn)(void *, int *);
typedef int (*nccl_count_fn)(void *, int *);
typedef int (*nccl_abort_fn)(void *);
struct Nccl {
  bool ok = false;
  nccl_async_err_fn async_err = nullptr;  // ncclCommGetAsyncError
  nccl_count_fn count = nullptr;          // ncclCommCount
  nccl_abort_fn abort = nullptr;          // ncclCommAbort
  nccl_get_uid_fn get_uid = nullptr;
  nccl_init_fn init = nullptr;
  nccl_destroy_fn destroy = nullptr;
  nccl_allgather_fn allgather = nullptr;
  nccl_allreduce_fn allreduce = nullptr;
  nccl_errstr_fn errstr = nullptr;
  char why[256] = "";
};
Nccl &nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *path = getenv("MOM_NCCL_LIB");
    void *h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(n.why, sizeof(n.why), "dlopen libnccl.so.2 failed: %s", dlerror());
      return;
    }
    n.get_uid = reinterpret_cast<nccl_get_uid_fn>(dlsym(h, "ncclGetUniqueId"));
    n.init = reinterpret_cast<nccl_init_fn>(dlsym(h, "ncclCommInitRank"));
    n.destroy = reinterpret_cast<nccl_destroy_fn>(dlsym(h, "ncclCommDestroy"));
    n.allgather = reinterpret_cast<nccl_allgather_fn>(dlsym(h, "ncclAllGather"));
    n.allreduce = reinterpret_cast<nccl_allreduce_fn>(dlsym(h, "ncclAllReduce"));
    n.errstr = reinterpret_cast<nccl_errstr_fn>(dlsym(h, "ncclGetErrorString"));
    n.async_err = reinterpret_cast<nccl_async_err_fn>(dlsym(h, "ncclCommGetAsyncError"));
    n.count = reinterpret_cast<nccl_count_fn>(dlsym(h, "ncclCommCount"));
    n.abort = reinterpret_cast<nccl_abort_fn>(dlsym(h, "ncclCommAbort"));
    n.ok = n.get_uid && n.init && n.destroy && n.allgather && n.allreduce && n.async_err && n.count && n.abort;
    if (!n.ok) snprintf(n.why, sizeof(n.why), "libnccl.so.2 lacks a required symbol");
  });
  return n;
}
mom_status_t nccl_fail(int rc, const char *what) {
  Nccl &n = nccl();
  return fail(MOM_ERR_NCCL, "%s: nccl error %d (%s)", what, rc, n.errstr ? n.errstr(rc) : "?");
}
// The communicator's asynchronous state (ncclCommGetAsyncError): a failed or aborted peer, a network or
// CUDA error inside an earlier collective.  ncclSuccess (0) and ncclInProgress (7) are healthy.
mom_status_t nccl_async_check(void *comm, const char *what) {
  Nccl &n = nccl();
  int st = 0;
  int rc = n.async_err(comm, &st);
  if (rc != 0) return nccl_fail(rc, "ncclCommGetAsyncError");
  if (st != 0 && st != 7) return nccl_fail(st, what);
  return MOM_OK;
}
}  // namespace

mom_status_t mom_nccl_check(void *comm) {
  g_err[0] = 0;
  if (!comm) return fail(MOM_ERR_INVALID_ARG, "mom_nccl_check: null comm");
  Nccl &n = nccl();
  if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
  return nccl_async_check(comm, "communicator in error state");
}

mom_status_t mom_nccl_comm_count(void *comm, int *nranks_out) {
  g_err[0] = 0;
  if (!comm || !nranks_out) return fail(MOM_ERR_INVALID_ARG, "mom_nccl_comm_count: null pointer");
  Nccl &n = nccl();
  if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
  int rc = n.count(comm, nranks_out);
  if (rc != 0) return nccl_fail(rc, "ncclCommCount");
  return MOM_OK;
}

mom_status_t mom_nccl_comm_abort(void *comm) {
  g_err[0] = 0;
  if (!comm) return fail(MOM_ERR_INVALID_ARG, "mom_nccl_comm_abort: null comm");
  Nccl &n = nccl();
  if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
  int rc = n.abort(comm);
  if (rc != 0) return nccl_fail(rc, "ncclCommAbort");
  return MOM_OK;
}

mom_status_t mom_nccl_get_unique_id(void *id_out) {
  g_err[0] = 0;
  if (!id_out) return fail(MOM_ERR_INVALID_ARG, "mom_nccl_get_unique_id: null pointer");
  Nccl &n = nccl();
  if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
  nccl_uid_t uid;
  int rc = n.get_uid(&uid);
  if (rc != 0) return nccl_fail(rc, "ncclGetUniqueId");
  memcpy(id_out, &uid, sizeof(uid));
  return MOM_OK;
}

mom_status_t mom_nccl_comm_init(void **comm_out, int nranks, const void *id, int rank) {
  g_err[0] = 0;
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(MOM_ERR_INVALID_ARG, "mom_nccl_comm_init: bad arguments");
  Nccl &n = nccl();
  if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
  nccl_uid_t uid;
  memcpy(&uid, id, sizeof(uid));
  int rc = n.init(comm_out, nranks, uid, rank);
  if (rc != 0) return nccl_fail(rc, "ncclCommInitRank");
  return MOM_OK;
}

mom_status_t mom_nccl_comm_destroy(void *comm) {
  g_err[0] = 0;
  if (!comm) return fail(MOM_ERR_INVALID_ARG, "mom_nccl_comm_destroy: null comm");
  Nccl &n = nccl();
  if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
  int rc = n.destroy(comm);
  if (rc != 0) return nccl_fail(rc, "ncclCommDestroy");
  return MOM_OK;
}

mom_status_t mom_allgather_rows(void *rows, int64_t rows_per_rank, int64_t hidden, mom_dtype_t dt, void *comm,
                                int rank, int nranks, mom_stream_t stream) {
  g_err[0] = 0;
  if (!rows || !comm || rows_per_rank < 1 || hidden < 1 || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(MOM_ERR_INVALID_ARG, "mom_allgather_rows: bad arguments");
  if (!valid_dtype(dt)) return fail(MOM_ERR_INVALID_ARG, "mom_allgather_rows: bad dtype");
  if (!aligned16(rows)) return fail(MOM_ERR_INVALID_ARG, "mom_allgather_rows: rows must be 16-byte aligned");
  Nccl &n = nccl();
  if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
  const size_t count = static_cast<size_t>(rows_per_rank) * static_cast<size_t>(hidden);
  const size_t w = dtype_bytes(dt);
  const int nccl_dtype = dt == MOM_BF16 ? 9 /* ncclBfloat16 */ : 7 /* ncclFloat32 */;
  const void *send = static_cast<const char *>(rows) + static_cast<size_t>(rank) * count * w;  // in-place
  NvtxRange nvtx("mom.allgather_rows");
  int rc = n.allgather(send, rows, count, nccl_dtype, comm, static_cast<cudaStream_t>(stream));
  if (rc != 0) return nccl_fail(rc, "ncclAllGather");
  return nccl_async_check(comm, "ncclAllGather (async)");
}

mom_status_t mom_nccl_barrier(void *comm, int32_t *scratch, mom_stream_t stream) {
  g_err[0] = 0;
  if (!comm || !scratch) return fail(MOM_ERR_INVALID_ARG, "mom_nccl_barrier: null pointer");
  Nccl &n = nccl();
  if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
  // a 1-element all-reduce on `stream`: no rank's later work starts before every rank's earlier
  // work on its stream (e.g. the peer stores of mom_mlp_minseq_fwd_gather) has completed
  NvtxRange nvtx("mom.nccl_barrier");
  int rc = n.allreduce(scratch, scratch, 1, 2 /* ncclInt32 */, 0 /* ncclSum */, comm, static_cast<cudaStream_t>(stream));
  if (rc != 0) return nccl_fail(rc, "ncclAllReduce(barrier)");
  return nccl_async_check(comm, "ncclAllReduce(barrier) (async)");
}

mom_status_t mom_argmax_allreduce(uint64_t *best_key, int32_t *argmax, void *comm, mom_stream_t stream) {
  g_err[0] = 0;
  if (!best_key || !argmax) return fail(MOM_ERR_INVALID_ARG, "mom_argmax_allreduce: null pointer");
  if ((reinterpret_cast<uintptr_t>(best_key) & 7) || (reinterpret_cast<uintptr_t>(argmax) & 3))
    return fail(MOM_ERR_INVALID_ARG, "mom_argmax_allreduce: misaligned pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (comm) {
    Nccl &n = nccl();
    if (!n.ok) return fail(MOM_ERR_NCCL, "%s", n.why);
    // u64 max over ranks of (order-preserving value << 32 | ~index): max logit, lowest index on ties
    int rc = n.allreduce(best_key, best_key, 1, 5 /* ncclUint64 */, 2 /* ncclMax */, comm, s);
    if (rc != 0) return nccl_fail(rc, "ncclAllReduce(max)");
    mom_status_t st = nccl_async_check(comm, "ncclAllReduce(max) (async)");
    if (st != MOM_OK) return st;
  }
  cudaError_t e = mom::launch_key_to_index(reinterpret_cast<const unsigned long long *>(best_key), argmax, s);
  if (e != cudaSuccess) return cuda_fail(e, "key to index");
  return MOM_OK;
}

}  // extern "C"
