// gemv.cu -- HBM-streaming kernels of MOM's last-token path (Alg. 1):
//   * last_token_mlp: O_last = residual + W_down (Swish(W_gate x) (.) W_up x)
//       kernel 1 streams W_gate and W_up (2*I*d*w bytes), keeps h in fp32;
//       kernel 2 streams W_down (d*I*w bytes), launched with PDL: it prefetches its W_down
//       rows into L2 while kernel 1 runs, then waits (griddepcontrol) and reads h via L1.
//   * lm_head: logits = W_head . rmsnorm(h) and the greedy token
//       streams W_head (V*d*w bytes) once; per-block packed (value, index) maxima, then a
//       one-block reduction.  Ties -> lowest index.
// All are bandwidth-bound: one warp per weight row, 16-byte coalesced vector loads issued
// in unrolled batches (8 x 16 B in flight per lane), fp32 accumulation, shuffle reductions.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace mom {
namespace gemv {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int UNROLL = 8;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint4 ld_stream(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// dot of 8 bf16 (one 16-B vector) with 8 fp32 from shared memory
__device__ __forceinline__ float dot8_bf16(const uint4 &w, const float *x) {
  const __nv_bfloat162 *w2 = reinterpret_cast<const __nv_bfloat162 *>(&w);
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 f = __bfloat1622float2(w2[e]);
    s = fmaf(f.x, x[2 * e], s);
    s = fmaf(f.y, x[2 * e + 1], s);
  }
  return s;
}
__device__ __forceinline__ float dot4_f32(const uint4 &w, const float *x) {
  float s = __uint_as_float(w.x) * x[0];
  s = fmaf(__uint_as_float(w.y), x[1], s);
  s = fmaf(__uint_as_float(w.z), x[2], s);
  s = fmaf(__uint_as_float(w.w), x[3], s);
  return s;
}

// Warp-level dot product of one weight row (n elements, 16-B aligned) with xs (smem fp32).
template <bool BF16>
__device__ __forceinline__ float row_dot(const void *wrow, const float *xs, int n, int lane) {
  constexpr int EPV = BF16 ? 8 : 4;  // elements per 16-B vector
  const int nvec = n / EPV;
  const uint4 *w = reinterpret_cast<const uint4 *>(wrow);
  float acc = 0.f;
  int v0 = 0;
  for (; v0 + 32 * UNROLL <= nvec; v0 += 32 * UNROLL) {
    uint4 buf[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) buf[u] = ld_stream(w + v0 + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int e = (v0 + u * 32 + lane) * EPV;
      acc += BF16 ? dot8_bf16(buf[u], xs + e) : dot4_f32(buf[u], xs + e);
    }
  }
  for (int v = v0 + lane; v < nvec; v += 32) {
    uint4 b = ld_stream(w + v);
    const int e = v * EPV;
    acc += BF16 ? dot8_bf16(b, xs + e) : dot4_f32(b, xs + e);
  }
  return warp_sum(acc);
}

// Two rows (gate and up) against the same smem vector, their loads interleaved so each lane
// keeps 2 * UNROLL 16-B requests in flight.
template <bool BF16>
__device__ __forceinline__ void row_dot2(const void *wrow0, const void *wrow1, const float *xs, int n, int lane,
                                         float &out0, float &out1) {
  constexpr int EPV = BF16 ? 8 : 4;
  const int nvec = n / EPV;
  const uint4 *w0 = reinterpret_cast<const uint4 *>(wrow0);
  const uint4 *w1 = reinterpret_cast<const uint4 *>(wrow1);
  float a0 = 0.f, a1 = 0.f;
  int v0 = 0;
  for (; v0 + 32 * UNROLL <= nvec; v0 += 32 * UNROLL) {
    uint4 b0[UNROLL], b1[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      b0[u] = ld_stream(w0 + v0 + u * 32 + lane);
      b1[u] = ld_stream(w1 + v0 + u * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int e = (v0 + u * 32 + lane) * EPV;
      a0 += BF16 ? dot8_bf16(b0[u], xs + e) : dot4_f32(b0[u], xs + e);
      a1 += BF16 ? dot8_bf16(b1[u], xs + e) : dot4_f32(b1[u], xs + e);
    }
  }
  for (int v = v0 + lane; v < nvec; v += 32) {
    const int e = v * EPV;
    const uint4 c0 = ld_stream(w0 + v), c1 = ld_stream(w1 + v);
    a0 += BF16 ? dot8_bf16(c0, xs + e) : dot4_f32(c0, xs + e);
    a1 += BF16 ? dot8_bf16(c1, xs + e) : dot4_f32(c1, xs + e);
  }
  out0 = warp_sum(a0);
  out1 = warp_sum(a1);
}

// Dot of one weight row with an fp32 vector read through the read-only/L1 path (no smem
// staging: every block starts streaming weights immediately).
template <bool BF16>
__device__ __forceinline__ float row_dot_gvec(const void *wrow, const float *__restrict__ hv, int n, int lane) {
  constexpr int EPV = BF16 ? 8 : 4;
  const int nvec = n / EPV;
  const uint4 *w = reinterpret_cast<const uint4 *>(wrow);
  float acc = 0.f;
  int v0 = 0;
  for (; v0 + 32 * UNROLL <= nvec; v0 += 32 * UNROLL) {
    uint4 buf[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) buf[u] = ld_stream(w + v0 + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int e = (v0 + u * 32 + lane) * EPV;
      float xv[EPV];
#pragma unroll
      for (int q = 0; q < EPV / 4; ++q) {
        const float4 f = __ldg(reinterpret_cast<const float4 *>(hv + e) + q);
        xv[4 * q] = f.x; xv[4 * q + 1] = f.y; xv[4 * q + 2] = f.z; xv[4 * q + 3] = f.w;
      }
      acc += BF16 ? dot8_bf16(buf[u], xv) : dot4_f32(buf[u], xv);
    }
  }
  for (int v = v0 + lane; v < nvec; v += 32) {
    const uint4 b = ld_stream(w + v);
    const int e = v * EPV;
    float xv[EPV];
#pragma unroll
    for (int q = 0; q < EPV / 4; ++q) {
      const float4 f = __ldg(reinterpret_cast<const float4 *>(hv + e) + q);
      xv[4 * q] = f.x; xv[4 * q + 1] = f.y; xv[4 * q + 2] = f.z; xv[4 * q + 3] = f.w;
    }
    acc += BF16 ? dot8_bf16(b, xv) : dot4_f32(b, xv);
  }
  return warp_sum(acc);
}

template <bool BF16>
__device__ __forceinline__ float load_elem(const void *p, size_t i) {
  if (BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i]);
  return reinterpret_cast<const float *>(p)[i];
}
template <bool BF16>
__device__ __forceinline__ void store_elem(void *p, size_t i, float v) {
  if (BF16)
    reinterpret_cast<__nv_bfloat16 *>(p)[i] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<float *>(p)[i] = v;
}

// Stage n elements (n % elements-per-16B == 0) of a bf16/fp32 vector into shared memory as fp32
// with independent 16-B loads (one round trip, not n/THREADS dependent ones); returns this
// thread's partial sum of squares.
template <bool BF16>
__device__ __forceinline__ float stage_vec(const void *src, float *dst, int n) {
  constexpr int EPV = BF16 ? 8 : 4;
  const uint4 *s = reinterpret_cast<const uint4 *>(src);
  float ss = 0.f;
#pragma unroll 4
  for (int v = threadIdx.x; v < n / EPV; v += THREADS) {
    const uint4 q = s[v];
    float f[EPV];
    if constexpr (BF16) {
      const __nv_bfloat162 *q2 = reinterpret_cast<const __nv_bfloat162 *>(&q);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 t = __bfloat1622float2(q2[e]);
        f[2 * e] = t.x;
        f[2 * e + 1] = t.y;
      }
    } else {
      f[0] = __uint_as_float(q.x); f[1] = __uint_as_float(q.y); f[2] = __uint_as_float(q.z); f[3] = __uint_as_float(q.w);
    }
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      dst[v * EPV + e] = f[e];
      ss = fmaf(f[e], f[e], ss);
    }
  }
  return ss;
}

// Programmatic dependent launch (PDL): the primary lets the next kernel in the stream launch
// early; the dependent prefetches its weight rows into L2 (they do not depend on the primary)
// and only then waits for the primary grid's results.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Prefetch (into L2) the weight rows this block's warps will stream: rows w, w + stride, ...
__device__ __forceinline__ void prefetch_my_rows(const void *base, size_t pitch, int rows, int max_rows_per_warp) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (lane < max_rows_per_warp) {
    const int r = w + lane * gridDim.x * WARPS;
    if (r < rows) prefetch_l2_bulk(static_cast<const char *>(base) + r * pitch, static_cast<uint32_t>(pitch));
  }
}

// h[j] = Swish(sum_k x_k Wg[j,k]) * (sum_k x_k Wu[j,k]), fp32.  Grid-stride over rows j.
template <bool BF16>
__global__ void __launch_bounds__(THREADS) gate_up_gemv(const void *__restrict__ x, const void *__restrict__ wg,
                                                        const void *__restrict__ wu, float *__restrict__ h, int d,
                                                        int I) {
  pdl_launch_dependents();  // the down GEMV may launch now and prefetch W_down
  extern __shared__ float xs[];
  stage_vec<BF16>(x, xs, d);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * WARPS + (threadIdx.x >> 5);
  const size_t pitch = static_cast<size_t>(d) * (BF16 ? 2 : 4);
  for (int j = w; j < I; j += gridDim.x * WARPS) {
    float g, u;
    row_dot2<BF16>(static_cast<const char *>(wg) + j * pitch, static_cast<const char *>(wu) + j * pitch, xs, d,
                   lane, g, u);
    if (lane == 0) h[j] = g / (1.0f + __expf(-g)) * u;
  }
}

// out[c] = residual[c] + sum_j h_j Wd[c,j].  h (fp32) read through L1 (no staging barrier).
template <bool BF16>
__global__ void __launch_bounds__(THREADS) down_gemv(const float *__restrict__ h, const void *__restrict__ wd,
                                                     const void *__restrict__ residual, void *__restrict__ out, int d,
                                                     int I, int prefetch_rows) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * WARPS + (threadIdx.x >> 5);
  const size_t pitch = static_cast<size_t>(I) * (BF16 ? 2 : 4);
  // W_down does not depend on h: pull this warp's rows towards L2 while gate/up still runs
  if ((pitch & 15) == 0 && prefetch_rows > 0) prefetch_my_rows(wd, pitch, d, prefetch_rows);
  pdl_launch_dependents();  // the LM head may launch early too
  pdl_wait();               // h (written by gate_up_gemv) is complete and visible from here on
  for (int c = w; c < d; c += gridDim.x * WARPS) {
    const float o = row_dot_gvec<BF16>(static_cast<const char *>(wd) + c * pitch, h, I, lane);
    if (lane == 0) {
      const float r = residual ? load_elem<BF16>(residual, c) : 0.f;
      store_elem<BF16>(out, c, r + o);
    }
  }
}

// Order-preserving map float -> uint32 (larger float -> larger key), then pack with the
// complemented index so that the u64 max picks the largest value and, among equal
// values, the LOWEST index.
__device__ __forceinline__ unsigned long long pack_key(float v, int idx) {
  uint32_t b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return (static_cast<unsigned long long>(b) << 32) | static_cast<uint32_t>(0xFFFFFFFFu - static_cast<uint32_t>(idx));
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  return v;
}

template <bool BF16>
__global__ void __launch_bounds__(THREADS) lm_head_gemv(const void *__restrict__ hin, const void *__restrict__ gain,
                                                        float eps, const void *__restrict__ w,
                                                        float *__restrict__ logits,
                                                        unsigned long long *__restrict__ partials, int d, int V,
                                                        int vocab_offset) {
  extern __shared__ float hs[];
  __shared__ float red[WARPS];
  __shared__ unsigned long long best_s[WARPS];
  pdl_wait();  // h comes from the previous kernel (PDL launch; a no-op without the attribute)
  // prologue: fp32 copy of h and (optionally) the final RMSNorm
  float ss = stage_vec<BF16>(hin, hs, d);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (gain) {
    ss = warp_sum(ss);
    if (lane == 0) red[wid] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int i = 0; i < WARPS; ++i) tot += red[i];
    const float inv = rsqrtf(tot / static_cast<float>(d) + eps);
    for (int k = threadIdx.x; k < d; k += THREADS) hs[k] = hs[k] * inv * load_elem<BF16>(gain, k);
  }
  __syncthreads();
  const int wglob = blockIdx.x * WARPS + wid;
  const size_t pitch = static_cast<size_t>(d) * (BF16 ? 2 : 4);
  unsigned long long best = 0ull;
  for (int v = wglob; v < V; v += gridDim.x * WARPS) {
    const float s = row_dot<BF16>(static_cast<const char *>(w) + v * pitch, hs, d, lane);
    if (lane == 0) {
      if (logits) logits[v] = s;
      const unsigned long long key = pack_key(s, v + vocab_offset);  // global vocab index
      best = key > best ? key : best;
    }
  }
  if (lane == 0) best_s[wid] = best;
  __syncthreads();
  if (wid == 0) {
    unsigned long long b = lane < WARPS ? best_s[lane] : 0ull;
    b = warp_max_u64(b);
    if (lane == 0) partials[blockIdx.x] = b;
  }
}

// Max over the per-block keys; writes the argmax (ties -> lowest index) and/or the packed key
// (the latter feeds the cross-rank u64 max of the vocab-sharded head, f2).
__global__ void argmax_reduce(const unsigned long long *__restrict__ partials, int n, int32_t *__restrict__ out,
                              unsigned long long *__restrict__ key_out) {
  __shared__ unsigned long long s[32];
  unsigned long long b = 0ull;
  for (int i = threadIdx.x; i < n; i += blockDim.x) b = partials[i] > b ? partials[i] : b;
  b = warp_max_u64(b);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x < 32) {
    b = threadIdx.x < blockDim.x / 32 ? s[threadIdx.x] : 0ull;
    b = warp_max_u64(b);
    if (threadIdx.x == 0) {
      if (out) out[0] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(b & 0xFFFFFFFFull));
      if (key_out) key_out[0] = b;
    }
  }
}

__global__ void key_to_index(const unsigned long long *__restrict__ key, int32_t *__restrict__ out) {
  out[0] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(key[0] & 0xFFFFFFFFull));
}

// Launch `kfn` on `stream` with programmatic stream serialization (PDL): it may start while
// the previous kernel in the stream is still running; it synchronises with griddepcontrol.wait.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kfn)(KArgs...), int blocks, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks, 1, 1);
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kfn, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_maybe_pdl(void (*kfn)(KArgs...), int blocks, size_t smem, cudaStream_t stream, bool pdl,
                                    Args... args) {
  if (pdl) return launch_pdl(kfn, blocks, smem, stream, args...);
  kfn<<<blocks, THREADS, smem, stream>>>(static_cast<KArgs>(args)...);
  return cudaGetLastError();
}

static int env_or(const char *name, int dflt) {
  const char *v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

template <typename K>
static cudaError_t set_smem(K kfn, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

}  // namespace gemv

cudaError_t launch_last_token_mlp(const void *x, const void *residual, const void *wg, const void *wu,
                                  const void *wd, void *out, float *h_ws, int d, int I, bool is_bf16, int num_sms,
                                  cudaStream_t stream) {
  using namespace gemv;
  const size_t smem1 = static_cast<size_t>(d) * sizeof(float);
  // Balanced single-wave grids: r = ceil(rows / resident warps) rows per warp, and just enough
  // warps that every warp gets r rows (or r - 1 for the last ones) -- no half-empty second round.
  auto balanced_blocks = [num_sms](int rows, int blocks_per_sm) {
    const int resident = num_sms * blocks_per_sm * WARPS;
    const int r = (rows + resident - 1) / resident;
    const int warps = (rows + r - 1) / r;
    return (warps + WARPS - 1) / WARPS;
  };
  const int blocks1 = balanced_blocks(I, 6);
  const int blocks2 = balanced_blocks(d, 6);
  const bool pdl = env_or("MOM_GEMV_PDL", 1) != 0;     // PDL launch of the down GEMV
  const int pf = env_or("MOM_GEMV_PREFETCH", 0);        // W_down rows per warp prefetched to L2 first
  cudaError_t e;
  if (is_bf16) {
    if ((e = set_smem(gate_up_gemv<true>, smem1)) != cudaSuccess) return e;
    gate_up_gemv<true><<<blocks1, THREADS, smem1, stream>>>(x, wg, wu, h_ws, d, I);
    if ((e = launch_maybe_pdl(down_gemv<true>, blocks2, 0, stream, pdl, h_ws, wd, residual, out, d, I, pf)) != cudaSuccess)
      return e;
  } else {
    if ((e = set_smem(gate_up_gemv<false>, smem1)) != cudaSuccess) return e;
    gate_up_gemv<false><<<blocks1, THREADS, smem1, stream>>>(x, wg, wu, h_ws, d, I);
    if ((e = launch_maybe_pdl(down_gemv<false>, blocks2, 0, stream, pdl, h_ws, wd, residual, out, d, I, pf)) != cudaSuccess)
      return e;
  }
  return cudaGetLastError();
}

size_t lm_head_partials(int num_sms) { return static_cast<size_t>(num_sms) * 4; }

cudaError_t launch_lm_head(const void *h, const void *gain, float eps, const void *w, float *logits,
                           int32_t *argmax, unsigned long long *key_out, int vocab_offset,
                           unsigned long long *partials, int d, int V, bool is_bf16, int num_sms,
                           cudaStream_t stream) {
  using namespace gemv;
  const size_t smem = static_cast<size_t>(d) * sizeof(float);
  int blocks = static_cast<int>(lm_head_partials(num_sms));
  const int need = (V + WARPS - 1) / WARPS;
  if (blocks > need) blocks = need;
  cudaError_t e;
  if (is_bf16) {
    if ((e = set_smem(lm_head_gemv<true>, smem)) != cudaSuccess) return e;
    e = launch_pdl(lm_head_gemv<true>, blocks, smem, stream, h, gain, eps, w, logits, partials, d, V, vocab_offset);
    if (e != cudaSuccess) return e;
  } else {
    if ((e = set_smem(lm_head_gemv<false>, smem)) != cudaSuccess) return e;
    e = launch_pdl(lm_head_gemv<false>, blocks, smem, stream, h, gain, eps, w, logits, partials, d, V, vocab_offset);
    if (e != cudaSuccess) return e;
  }
  argmax_reduce<<<1, 1024, 0, stream>>>(partials, blocks, argmax, key_out);
  return cudaGetLastError();
}

cudaError_t launch_key_to_index(const unsigned long long *key, int32_t *argmax, cudaStream_t stream) {
  gemv::key_to_index<<<1, 1, 0, stream>>>(key, argmax);
  return cudaGetLastError();
}

}  // namespace mom
