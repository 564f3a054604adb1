// gemv.cu -- HBM-streaming kernels of MOM's last-token path (Alg. 1):
//   * last_token_mlp: O_last = residual + W_down (Swish(W_gate x) (.) W_up x)
//       kernel 1 streams W_gate and W_up (2*I*d*w bytes), keeps h in fp32;
//       kernel 2 streams W_down (d*I*w bytes), launched with PDL: it prefetches its W_down
//       rows into L2 while kernel 1 runs, then waits (griddepcontrol) and reads h via L1.
//   * lm_head: logits = W_head . rmsnorm(h) and the greedy token
//       streams W_head (V*d*w bytes) once; per-block packed (value, index) maxima, then a
//       one-block reduction.  Ties -> lowest index.
// All are bandwidth-bound: a warp streams a few weight rows at once (rows_dot: the vector
// slice each lane needs is read once and reused for every row, so shared-memory / L1 reads do not
// limit the rate when the SM clock is low under the power cap), 16-byte coalesced vector loads,
// 8 x 16 B in flight per lane, fp32 accumulation, shuffle reductions.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace mom {
namespace gemv {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;

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

// R consecutive rows of each of NM weight matrices (same row pitch `pitch` bytes) against the
// same fp32 vector x (shared memory, or global through L1 when XG): each lane reads its slice of x
// ONCE per step and uses it for all NM * R rows (NM * R x fewer x reads per weight byte than
// row_dot), with NM * R * UNROLL_R 16-B weight loads in flight.  Rows >= nrows are clamped to
// the last valid row (their results are discarded).  Per row, the summation order is fixed
// (ascending 16-B vector index per lane, then the warp_sum butterfly) and does not depend on R,
// NM or the grid, so a row's result is the same whichever warp computes it (f2's shards).
template <bool BF16, int NM, int R, bool XG, int UNROLL_R = 2>
__device__ __forceinline__ void rows_dot(const char *const (&base)[NM], size_t pitch, int nrows,
                                         const float *__restrict__ x, int n, int lane, float (&out)[NM][R]) {
  constexpr int EPV = BF16 ? 8 : 4;
  const int nvec = n / EPV;
  int off[R];  // row offsets in 16-B vectors (32-bit: fewer registers than NM * R pointers)
#pragma unroll
  for (int r = 0; r < R; ++r) off[r] = (r < nrows ? r : nrows - 1) * static_cast<int>(pitch / 16);
  float acc[NM][R];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[m][r] = 0.f;
  auto load_x = [&](int e, float (&xv)[EPV]) {
#pragma unroll
    for (int q = 0; q < EPV / 4; ++q) {
      const float4 f = XG ? __ldg(reinterpret_cast<const float4 *>(x + e) + q) : reinterpret_cast<const float4 *>(x + e)[q];
      xv[4 * q] = f.x; xv[4 * q + 1] = f.y; xv[4 * q + 2] = f.z; xv[4 * q + 3] = f.w;
    }
  };
  int v0 = 0;
  for (; v0 + 32 * UNROLL_R <= nvec; v0 += 32 * UNROLL_R) {
    uint4 buf[UNROLL_R][NM][R];
#pragma unroll
    for (int u = 0; u < UNROLL_R; ++u)
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int r = 0; r < R; ++r)
          buf[u][m][r] = ld_stream(reinterpret_cast<const uint4 *>(base[m]) + off[r] + v0 + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < UNROLL_R; ++u) {
      float xv[EPV];
      load_x((v0 + u * 32 + lane) * EPV, xv);
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[m][r] += BF16 ? dot8_bf16(buf[u][m][r], xv) : dot4_f32(buf[u][m][r], xv);
    }
  }
  for (int v = v0 + lane; v < nvec; v += 32) {
    float xv[EPV];
    load_x(v * EPV, xv);
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint4 b = ld_stream(reinterpret_cast<const uint4 *>(base[m]) + off[r] + v);
        acc[m][r] += BF16 ? dot8_bf16(b, xv) : dot4_f32(b, xv);
      }
  }
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) out[m][r] = warp_sum(acc[m][r]);
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
// Prefetch (into L2) the first `bytes` of the R consecutive weight rows this warp streams first
// (rows w*R .. w*R+R-1): issued before griddepcontrol.wait, so they arrive while the primary grid
// drains and the warp's first loads hit L2.
__device__ __forceinline__ void prefetch_first_rows(const void *base, size_t pitch, int rows, int R, uint32_t bytes) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int r = w * R + lane;
  if (lane < R && r < rows) prefetch_l2_bulk(static_cast<const char *>(base) + r * pitch, bytes);
}

// h[j] = Swish(sum_k x_k Wg[j,k]) * (sum_k x_k Wu[j,k]), fp32.  Warp-stride over groups of R
// rows j (gate and up rows of each j streamed together).
// norm_eps >= 0: the f3 form -- x is first scaled by r = 1/sqrt(mean(x^2) + eps) (the gain is
// folded into W_gate / W_up by the caller), i.e. h = Swish(Wg' (r x)) (.) (Wu' (r x)).
template <bool BF16, int R, int U = 2, int MINB = 4>
__global__ void __launch_bounds__(THREADS, MINB) gate_up_gemv(const void *__restrict__ x, const void *__restrict__ wg,
                                                           const void *__restrict__ wu, float *__restrict__ h, int d,
                                                           int I, float norm_eps) {
  pdl_launch_dependents();  // the down GEMV may launch now
  // launched with PDL after the producer of x (the last mini-sequence layer's phase B): the CTAs
  // become resident as that grid's CTAs retire, and wait here for its results
  pdl_wait();
  extern __shared__ float xs[];
  __shared__ float red[WARPS];
  float ss = stage_vec<BF16>(x, xs, d);
  if (norm_eps >= 0.f) {  // fold RMSNorm: the sum of squares came with the staging pass
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int i = 0; i < WARPS; ++i) tot += red[i];
    const float inv = rsqrtf(tot / static_cast<float>(d) + norm_eps);
    for (int k = threadIdx.x; k < d; k += THREADS) xs[k] *= inv;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * WARPS + (threadIdx.x >> 5);
  const size_t pitch = static_cast<size_t>(d) * (BF16 ? 2 : 4);
  for (int j0 = w * R; j0 < I; j0 += gridDim.x * WARPS * R) {
    float gu[2][R];
    const char *const base[2] = {static_cast<const char *>(wg) + j0 * pitch, static_cast<const char *>(wu) + j0 * pitch};
    rows_dot<BF16, 2, R, false, U>(base, pitch, I - j0, xs, d, lane, gu);
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (j0 + r < I) h[j0 + r] = gu[0][r] / (1.0f + __expf(-gu[0][r])) * gu[1][r];
    }
  }
}

// out[c] = residual[c] + sum_j h_j Wd[c,j].  h (fp32) read through L1 (no staging barrier).
template <bool BF16, int R, int U = 2, int MINB = 4>
__global__ void __launch_bounds__(THREADS, MINB) down_gemv(const float *__restrict__ h, const void *__restrict__ wd,
                                                        const void *__restrict__ residual, void *__restrict__ out,
                                                        int d, int I, int prefetch_bytes) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * WARPS + (threadIdx.x >> 5);
  const size_t pitch = static_cast<size_t>(I) * (BF16 ? 2 : 4);
  // W_down does not depend on h: pull the head of this warp's first rows towards L2 while gate/up
  // drains (prefetch_bytes per row, 16-B multiple, <= the row)
  if (prefetch_bytes > 0) prefetch_first_rows(wd, pitch, d, R, static_cast<uint32_t>(prefetch_bytes));
  pdl_launch_dependents();  // the LM head may launch early too
  pdl_wait();               // h (written by gate_up_gemv) is complete and visible from here on
  for (int c0 = w * R; c0 < d; c0 += gridDim.x * WARPS * R) {
    float o[1][R];
    const char *const base[1] = {static_cast<const char *>(wd) + c0 * pitch};
    rows_dot<BF16, 1, R, true, U>(base, pitch, d - c0, h, I, lane, o);
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (c0 + r < d) {
          const float rv = residual ? load_elem<BF16>(residual, c0 + r) : 0.f;
          store_elem<BF16>(out, c0 + r, rv + o[0][r]);
        }
      }
    }
  }
}

// K-split down GEMV (bf16): KS consecutive warps of a block share R rows; warp q sums the 16-B vectors
// of its slice [q n / KS, (q+1) n / KS) of each row, and the KS partial sums are added in q order through
// shared memory (a fixed order: deterministic).  Each warp's chain of dependent loads is KS times
// shorter and KS times more warps stream at once than in down_gemv, for the same rows.  The loop trip
// count is uniform across the block (block-wide barriers inside).
template <int R, int U, int KS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) down_gemv_ks(const float *__restrict__ h, const void *__restrict__ wd,
                                                           const void *__restrict__ residual, void *__restrict__ out,
                                                           int d, int I) {
  constexpr int GPB = WARPS / KS;  // row groups per block
  __shared__ float part[WARPS][R];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int grp = wid / KS, q = wid % KS;
  const int nvec = I / 8;
  const int v_lo = q * nvec / KS, v_hi = (q + 1) * nvec / KS;
  const size_t pitch = static_cast<size_t>(I) * 2;
  const int stride = gridDim.x * GPB * R;
  const int iters = (d + stride - 1) / stride;
  pdl_launch_dependents();  // the LM head may launch early too
  pdl_wait();               // h (written by gate_up_gemv) is complete and visible from here on
  for (int it = 0; it < iters; ++it) {
    const int c0 = it * stride + (blockIdx.x * GPB + grp) * R;
    if (c0 < d) {
      float o[1][R];
      const char *const base[1] = {static_cast<const char *>(wd) + c0 * pitch + static_cast<size_t>(v_lo) * 16};
      rows_dot<true, 1, R, true, U>(base, pitch, d - c0, h + 8 * v_lo, (v_hi - v_lo) * 8, lane, o);
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) part[wid][r] = o[0][r];
      }
    }
    __syncthreads();
    if (q == 0 && lane == 0 && c0 < d) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (c0 + r < d) {
          float t = 0.f;
#pragma unroll
          for (int k = 0; k < KS; ++k) t += part[grp * KS + k][r];
          const float rv = residual ? __bfloat162float(static_cast<const __nv_bfloat16 *>(residual)[c0 + r]) : 0.f;
          static_cast<__nv_bfloat16 *>(out)[c0 + r] = __float2bfloat16_rn(rv + t);
        }
      }
    }
    __syncthreads();
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

template <bool BF16, int R, int U>
__global__ void __launch_bounds__(THREADS, 4) lm_head_gemv(const void *__restrict__ hin, const void *__restrict__ gain,
                                                        float eps, const void *__restrict__ w,
                                                        float *__restrict__ logits,
                                                        unsigned long long *__restrict__ partials, int d, int V,
                                                        int vocab_offset) {
  extern __shared__ float hs[];
  __shared__ float red[WARPS];
  __shared__ unsigned long long best_s[WARPS];
  pdl_wait();  // h comes from the previous kernel (PDL launch; a no-op without the attribute)
  pdl_launch_dependents();  // argmax_reduce may launch now (it waits for this grid's partials)
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
  // warp-stride over groups of R consecutive rows
  for (int v0 = wglob * R; v0 < V; v0 += gridDim.x * WARPS * R) {
    float s[1][R];
    const char *const base[1] = {static_cast<const char *>(w) + v0 * pitch};
    rows_dot<BF16, 1, R, false, U>(base, pitch, V - v0, hs, d, lane, s);
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (v0 + r < V) {
          if (logits) logits[v0 + r] = s[0][r];
          const unsigned long long key = pack_key(s[0][r], v0 + r + vocab_offset);  // global vocab index
          best = key > best ? key : best;
        }
      }
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
  pdl_wait();  // launched with PDL behind lm_head_gemv: its partials are complete from here on
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
static cudaError_t launch_maybe_pdl_threads(void (*kfn)(KArgs...), int blocks, int threads, cudaStream_t stream,
                                            bool pdl, Args... args) {
  if (!pdl) {
    kfn<<<blocks, threads, 0, stream>>>(static_cast<KArgs>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
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

template <bool BF16, int RG, int UG, int MG, int RD, int UD, int MD>
static cudaError_t last_token_pair(const void *x, const void *residual, const void *wg, const void *wu, const void *wd,
                                   void *out, float *h_ws, int d, int I, int num_sms, cudaStream_t stream,
                                   float norm_eps) {
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
  const int blocks1 = balanced_blocks((I + RG - 1) / RG, MG);
  const int blocks2 = balanced_blocks((d + RD - 1) / RD, MD);
  const bool pdl = env_or("MOM_GEMV_PDL", 1) != 0;     // PDL launches of both GEMVs
  // KB of each warp's first W_down rows prefetched to L2 before waiting for gate/up (0 = off)
  int pf = env_or("MOM_GEMV_PREFETCH", 0) * 1024;
  const int row_bytes = I * (BF16 ? 2 : 4);
  if (pf > row_bytes) pf = row_bytes;
  pf &= ~15;
  cudaError_t e;
  if ((e = set_smem(gate_up_gemv<BF16, RG, UG, MG>, smem1)) != cudaSuccess) return e;
  if ((e = launch_maybe_pdl(gate_up_gemv<BF16, RG, UG, MG>, blocks1, smem1, stream, pdl, x, wg, wu, h_ws, d, I,
                            norm_eps)) != cudaSuccess)
    return e;
  if ((e = launch_maybe_pdl(down_gemv<BF16, RD, UD, MD>, blocks2, 0, stream, pdl, h_ws, wd, residual, out, d, I, pf)) !=
      cudaSuccess)
    return e;
  return cudaGetLastError();
}

cudaError_t launch_last_token_mlp(const void *x, const void *residual, const void *wg, const void *wu,
                                  const void *wd, void *out, float *h_ws, int d, int I, bool is_bf16, int num_sms,
                                  cudaStream_t stream, float norm_eps) {
  // Default (MOM_GEMV_VARIANT=5, bf16): gate/up 2 rows x 2 x 2 loads in flight at 4 blocks/SM, down
  // K-split over 2 warps per 2-row group (profiles/r2_gemv_ksplit_ab.txt).  Variants 0-3: the
  // un-split down GEMV with (rows per warp step, 16-B loads in flight per row, min blocks per SM) =
  // (2, 2, 4) / (2, 4, 2) / (2, 8, 2) -- 2 x 2 at 4/SM had 4 MB in flight and was latency-bound at
  // ~3.5 TB/s (profiles/r1_gemv_variants.txt).  fp32: the pair with (2, 2, 4).
  if (!is_bf16) return last_token_pair<false, 2, 2, 4, 2, 2, 4>(x, residual, wg, wu, wd, out, h_ws, d, I, num_sms, stream, norm_eps);
  const int variant = gemv::env_or("MOM_GEMV_VARIANT", 5);
  if (is_bf16 && (variant == 5 || variant == 6) && I / 8 >= 4) {
    // gate/up as variant 2; down K-split over KS = 2 (5) or 4 (6) warps per row group
    using namespace gemv;
    const size_t smem1 = static_cast<size_t>(d) * sizeof(float);
    cudaError_t e;
    if ((e = set_smem(gate_up_gemv<true, 2, 2, 4>, smem1)) != cudaSuccess) return e;
    const int resident = num_sms * 4 * WARPS;
    const int groups = (I + 1) / 2, r = (groups + resident - 1) / resident;
    const int blocks1 = ((groups + r - 1) / r + WARPS - 1) / WARPS;
    const bool pdl = env_or("MOM_GEMV_PDL", 1) != 0;
    if ((e = launch_maybe_pdl(gate_up_gemv<true, 2, 2, 4>, blocks1, smem1, stream, pdl, x, wg, wu, h_ws, d, I,
                              norm_eps)) != cudaSuccess)
      return e;
    // single balanced wave: rows per iteration = blocks * (WARPS / KS) * 2 >= d when it fits
    const int ks = variant == 5 ? 2 : 4;
    const int rows_per_block = (WARPS / ks) * 2;
    int blocks2 = (d + rows_per_block - 1) / rows_per_block;
    if (blocks2 > num_sms * 4) blocks2 = num_sms * 4;
    if (variant == 5)
      return launch_maybe_pdl(down_gemv_ks<2, 4, 2, 4>, blocks2, 0, stream, pdl, static_cast<const float *>(h_ws), wd,
                              residual, out, d, I);
    return launch_maybe_pdl(down_gemv_ks<2, 4, 4, 4>, blocks2, 0, stream, pdl, static_cast<const float *>(h_ws), wd,
                            residual, out, d, I);
  }
  if (variant == 0)
    return last_token_pair<true, 2, 2, 4, 2, 2, 4>(x, residual, wg, wu, wd, out, h_ws, d, I, num_sms, stream, norm_eps);
  // deeper per-lane load queues (same per-row summation order: bit-neutral): down 8 loads in flight
  // per row (2, the default: 69 vs 70 us inside the bench step, profiles/r2_gemv_inbench_ab2.txt), and
  // gate/up 4 per row at 2 blocks/SM as well (3)
  if (variant == 2)
    return last_token_pair<true, 2, 2, 4, 2, 8, 2>(x, residual, wg, wu, wd, out, h_ws, d, I, num_sms, stream, norm_eps);
  if (variant == 3)
    return last_token_pair<true, 2, 4, 2, 2, 8, 2>(x, residual, wg, wu, wd, out, h_ws, d, I, num_sms, stream, norm_eps);
  return last_token_pair<true, 2, 2, 4, 2, 4, 2>(x, residual, wg, wu, wd, out, h_ws, d, I, num_sms, stream, norm_eps);
}

size_t lm_head_partials(int num_sms) { return static_cast<size_t>(num_sms) * 4; }

cudaError_t launch_lm_head(const void *h, const void *gain, float eps, const void *w, float *logits,
                           int32_t *argmax, unsigned long long *key_out, int vocab_offset,
                           unsigned long long *partials, int d, int V, bool is_bf16, int num_sms,
                           cudaStream_t stream) {
  using namespace gemv;
  const size_t smem = static_cast<size_t>(d) * sizeof(float);
  // 4 rows per warp step (x reused from registers across them) x 2 16-B loads in flight per row
  // (measured: 2 rows x 4 loads is equivalent, tools/head_variants.sh)
  constexpr int R = 4, U = 2;
  // balanced single wave (4 blocks per SM resident): every warp gets r or r - 1 row groups
  const int groups = (V + R - 1) / R;
  const int resident = static_cast<int>(lm_head_partials(num_sms)) * WARPS;
  const int r = (groups + resident - 1) / resident;
  const int blocks = ((groups + r - 1) / r + WARPS - 1) / WARPS;
  cudaError_t e;
  if (is_bf16) {
    if ((e = set_smem(lm_head_gemv<true, R, U>, smem)) != cudaSuccess) return e;
    e = launch_pdl(lm_head_gemv<true, R, U>, blocks, smem, stream, h, gain, eps, w, logits, partials, d, V, vocab_offset);
  } else {
    if ((e = set_smem(lm_head_gemv<false, R, U>, smem)) != cudaSuccess) return e;
    e = launch_pdl(lm_head_gemv<false, R, U>, blocks, smem, stream, h, gain, eps, w, logits, partials, d, V, vocab_offset);
  }
  if (e != cudaSuccess) return e;
  // PDL: the reduction's launch overlaps the head's tail; it waits in griddepcontrol.wait
  return launch_maybe_pdl_threads(argmax_reduce, 1, 1024, stream, env_or("MOM_GEMV_PDL", 1) != 0, partials, blocks,
                                  argmax, key_out);
}

cudaError_t launch_key_to_index(const unsigned long long *key, int32_t *argmax, cudaStream_t stream) {
  gemv::key_to_index<<<1, 1, 0, stream>>>(key, argmax);
  return cudaGetLastError();
}

}  // namespace mom
