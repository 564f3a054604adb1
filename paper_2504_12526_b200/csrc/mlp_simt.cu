// mlp_simt.cu -- fp32 SIMT kernels for the mini-sequence SwiGLU MLP (MOM_F32 dtype).
//
// The fp32 variant exists for the small parity configuration (BASELINE config 1: hidden 256,
// intermediate 688): tensor-core TF32 cannot meet the 1e-4 fp32 tolerance, so this path uses
// FFMA with fp32 accumulation.  Same Phase A / Phase B split as the tcgen05 path:
//   Phase A: H = Swish(X Wg^T) (.) (X Wu^T)
//   Phase B: out = residual + H Wd^T
// 64 x 64 output tiles, K staged through shared memory 16 at a time, 256 threads with a
// 4 x 4 register micro-tile each.  Each output sums K in ascending order, so results do not
// depend on the mini-sequence partition.
#include <cuda_runtime.h>

#include "kernels.h"

namespace mom {
namespace simt {

constexpr int TM = 64, TN = 64, TK = 16, THREADS = 256;

// acc[i][j] += sum_k A[m0+ty*4+i, k] * B[n0+tx*4+j, k], A: [rows, K], B: [N, K] (both K-contiguous)
template <bool DUAL>
__global__ void __launch_bounds__(THREADS) gemm_nt_kernel(const float *__restrict__ A, const float *__restrict__ B0,
                                                          const float *__restrict__ B1,
                                                          const float *__restrict__ residual,
                                                          float *__restrict__ out, int rows, int N, int K) {
  __shared__ float sA[TK][TM + 4];
  __shared__ float sB0[TK][TN + 4];
  __shared__ float sB1[DUAL ? TK : 1][TN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc0[4][4] = {}, acc1[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    // each thread loads 4 elements of each 64 x 16 tile
    for (int e = tid; e < TM * TK; e += THREADS) {
      const int r = e / TK, kk = e % TK;
      const int gr = m0 + r, gk = k0 + kk;
      sA[kk][r] = (gr < rows && gk < K) ? A[(size_t)gr * K + gk] : 0.f;
      const int gn = n0 + r;
      sB0[kk][r] = (gn < N && gk < K) ? B0[(size_t)gn * K + gk] : 0.f;
      if (DUAL) sB1[kk][r] = (gn < N && gk < K) ? B1[(size_t)gn * K + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b0[4], b1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        b0[j] = sB0[kk][tx * 4 + j];
        if (DUAL) b1[j] = sB1[kk][tx * 4 + j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc0[i][j] = fmaf(a[i], b0[j], acc0[i][j]);
          if (DUAL) acc1[i][j] = fmaf(a[i], b1[j], acc1[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + ty * 4 + i;
    if (r >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
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
