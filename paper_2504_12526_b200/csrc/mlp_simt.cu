// mlp_simt.cu -- fp32 SIMT kernels for the mini-sequence SwiGLU MLP (MOM_F32 dtype).
//
// The fp32 variant exists for the small parity configuration (BASELINE config 1: hidden 256,
// intermediate 688): tensor-core TF32 cannot meet the 1e-4 fp32 tolerance, so this path uses
// FFMA with fp32 accumulation.  Same Phase A / Phase B split as the tcgen05 path:
//   Phase A: H = Swish(X Wg^T) (.) (X Wu^T)
//   Phase B: out = residual + H Wd^T
// 32 x 32 output tiles, K staged through double-buffered shared memory 32 at a time, 256 threads
// with a 2 x 2 register micro-tile each.  Each output sums K in ascending order (one fma chain), so
// results do not depend on the mini-sequence partition.
#include <cuda_runtime.h>

#include "kernels.h"

namespace mom {
namespace simt {

// 32 x 32 output tiles (4x more blocks than 64 x 64 at config 1's 256-row mini-sequences, where the grid
// had only 16-44 blocks), K staged through shared memory 32 at a time with the next K tile prefetched into
// registers while the current one is consumed (the per-K-step global latency is hidden), 256 threads
// with a 2 x 2 register micro-tile.  Every output still sums K in ascending order with one fma chain.
constexpr int TM = 32, TN = 32, TK = 32, THREADS = 256;

// acc[i][j] += sum_k A[m0+ty*2+i, k] * B[n0+tx*2+j, k], A: [rows, K], B: [N, K] (both K-contiguous,
// K % 4 == 0: the fp32 row pitch is a multiple of 16 bytes)
template <bool DUAL>
__global__ void __launch_bounds__(THREADS) gemm_nt_kernel(const float *__restrict__ A, const float *__restrict__ B0,
                                                          const float *__restrict__ B1,
                                                          const float *__restrict__ residual,
                                                          float *__restrict__ out, int rows, int N, int K) {
  __shared__ float sA[2][TK][TM + 4];
  __shared__ float sB0[2][TK][TN + 4];
  __shared__ float sB1[DUAL ? 2 : 1][DUAL ? TK : 1][TN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  // loader mapping: one float4 of A, B0 (and B1) per thread per K tile: row lr, K quad lq
  const int lr = tid / (TK / 4), lq = tid % (TK / 4);
  float4 ra, rb0, rb1;
  auto load = [&](int k0) {
    const int gk = k0 + 4 * lq;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    ra = (m0 + lr < rows && gk < K) ? *reinterpret_cast<const float4 *>(A + (size_t)(m0 + lr) * K + gk) : z;
    rb0 = (n0 + lr < N && gk < K) ? *reinterpret_cast<const float4 *>(B0 + (size_t)(n0 + lr) * K + gk) : z;
    if (DUAL) rb1 = (n0 + lr < N && gk < K) ? *reinterpret_cast<const float4 *>(B1 + (size_t)(n0 + lr) * K + gk) : z;
  };
  auto stash = [&](int buf) {
    sA[buf][4 * lq + 0][lr] = ra.x; sA[buf][4 * lq + 1][lr] = ra.y; sA[buf][4 * lq + 2][lr] = ra.z; sA[buf][4 * lq + 3][lr] = ra.w;
    sB0[buf][4 * lq + 0][lr] = rb0.x; sB0[buf][4 * lq + 1][lr] = rb0.y; sB0[buf][4 * lq + 2][lr] = rb0.z; sB0[buf][4 * lq + 3][lr] = rb0.w;
    if (DUAL) {
      sB1[buf][4 * lq + 0][lr] = rb1.x; sB1[buf][4 * lq + 1][lr] = rb1.y; sB1[buf][4 * lq + 2][lr] = rb1.z; sB1[buf][4 * lq + 3][lr] = rb1.w;
    }
  };
  float acc0[2][2] = {}, acc1[2][2] = {};
  load(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += TK) {
    const bool more = k0 + TK < K;
    if (more) load(k0 + TK);  // in flight while this tile is consumed
    const int kn = K - k0 < TK ? K - k0 : TK;  // no padded terms: the fma chain is exactly K long
#pragma unroll 8
    for (int kk = 0; kk < kn; ++kk) {
      const float a0 = sA[buf][kk][ty * 2], a1 = sA[buf][kk][ty * 2 + 1];
      const float b00 = sB0[buf][kk][tx * 2], b01 = sB0[buf][kk][tx * 2 + 1];
      acc0[0][0] = fmaf(a0, b00, acc0[0][0]);
      acc0[0][1] = fmaf(a0, b01, acc0[0][1]);
      acc0[1][0] = fmaf(a1, b00, acc0[1][0]);
      acc0[1][1] = fmaf(a1, b01, acc0[1][1]);
      if (DUAL) {
        const float b10 = sB1[buf][kk][tx * 2], b11 = sB1[buf][kk][tx * 2 + 1];
        acc1[0][0] = fmaf(a0, b10, acc1[0][0]);
        acc1[0][1] = fmaf(a0, b11, acc1[0][1]);
        acc1[1][0] = fmaf(a1, b10, acc1[1][0]);
        acc1[1][1] = fmaf(a1, b11, acc1[1][1]);
      }
    }
    if (more) stash(buf ^ 1);  // the other buffer: last read before the previous barrier
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = m0 + ty * 2 + i;
    if (r >= rows) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = n0 + tx * 2 + j;
      if (c >= N) continue;
      float v;
      if (DUAL) {
        const float g = acc0[i][j], u = acc1[i][j];
        v = g / (1.0f + expf(-g)) * u;  // Swish(g) * u
      } else {
        v = acc0[i][j] + (residual ? residual[(size_t)r * N + c] : 0.f);
      }
      out[(size_t)r * N + c] = v;
    }
  }
}

}  // namespace simt

cudaError_t launch_phase_a_f32(const float *x, const float *wg, const float *wu, float *h, int rows, int d, int I,
                               cudaStream_t stream) {
  dim3 grid((I + simt::TN - 1) / simt::TN, (rows + simt::TM - 1) / simt::TM);
  simt::gemm_nt_kernel<true><<<grid, simt::THREADS, 0, stream>>>(x, wg, wu, nullptr, h, rows, I, d);
  return cudaGetLastError();
}

cudaError_t launch_phase_b_f32(const float *h, const float *wd, const float *residual, float *out, int rows, int d,
                               int I, cudaStream_t stream) {
  dim3 grid((d + simt::TN - 1) / simt::TN, (rows + simt::TM - 1) / simt::TM);
  simt::gemm_nt_kernel<false><<<grid, simt::THREADS, 0, stream>>>(h, wd, nullptr, residual, out, rows, d, I);
  return cudaGetLastError();
}

}  // namespace mom
