// norm.cu -- the per-layer RMSNorm folded into the mini-sequence MLP.
//
// A Llama block's MLP half is  out = x + MLP(RMSNorm(x) (.) g)  (SPEC S:260 pre-norm block;
// RMSNorm S:126).  With RMSNorm(x)_k = x_k * r, r = 1/sqrt(mean(x^2) + eps):
//     (RMSNorm(x) (.) g) W^T = r * x (W diag(g))^T
// so the gain is folded into W_gate / W_up once (fold_gain_kernel, at weight-load time) and the
// per-row scale r is applied to the fp32 gate/up accumulators in the phase-A epilogue.  The only
// extra pass is row_inv_rms_kernel over one mini-sequence's rows (C * d * w bytes, L2-resident
// for the phase-A launch that follows); the normed [S, d] tensor is never written.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace mom {
namespace norm {

// w_out[j, k] = round_bf16(w[j, k] * g[k]); 8 elements (16 B) per thread-iteration.
__global__ void fold_gain_kernel(const __nv_bfloat16 *__restrict__ w, const __nv_bfloat16 *__restrict__ g,
                                 __nv_bfloat16 *__restrict__ out, int64_t rows, int64_t cols) {
  const int64_t nvec = rows * cols / 8;
  const int64_t cvec = cols / 8;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c8 = (v % cvec) * 8;
    uint4 wv = reinterpret_cast<const uint4 *>(w)[v];
    uint4 gv = *reinterpret_cast<const uint4 *>(g + c8);
    const __nv_bfloat162 *w2 = reinterpret_cast<const __nv_bfloat162 *>(&wv);
    const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gv);
    uint4 o;
    __nv_bfloat162 *o2 = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 a = __bfloat1622float2(w2[e]), b = __bfloat1622float2(g2[e]);
      o2[e] = __floats2bfloat162_rn(a.x * b.x, a.y * b.y);
    }
    reinterpret_cast<uint4 *>(out)[v] = o;
  }
}

// r[row] = 1 / sqrt(mean_k x[row, k]^2 + eps), fp32; one warp per row, 16-B loads.
__global__ void row_inv_rms_kernel(const __nv_bfloat16 *__restrict__ x, float *__restrict__ r, int rows, int d,
                                   float eps) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int row = warp; row < rows; row += nwarps) {
    const uint4 *xr = reinterpret_cast<const uint4 *>(x + static_cast<size_t>(row) * d);
    float ss = 0.f;
    for (int v = lane; v < d / 8; v += 32) {
      uint4 q = xr[v];
      const __nv_bfloat162 *q2 = reinterpret_cast<const __nv_bfloat162 *>(&q);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(q2[e]);
        ss = fmaf(f.x, f.x, ss);
        ss = fmaf(f.y, f.y, ss);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) r[row] = rsqrtf(ss / static_cast<float>(d) + eps);
  }
}

}  // namespace norm

cudaError_t launch_fold_gain(const __nv_bfloat16 *w, const __nv_bfloat16 *g, __nv_bfloat16 *out, int64_t rows,
                             int64_t cols, int num_sms, cudaStream_t stream) {
  const int64_t nvec = rows * cols / 8;
  int64_t blocks = (nvec + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  if (blocks < 1) blocks = 1;
  norm::fold_gain_kernel<<<(unsigned)blocks, 256, 0, stream>>>(w, g, out, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_row_inv_rms(const __nv_bfloat16 *x, float *r, int rows, int d, float eps, int num_sms,
                               cudaStream_t stream) {
  int blocks = (rows + 7) / 8;  // 8 warps per block, one row per warp
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  if (blocks < 1) blocks = 1;
  norm::row_inv_rms_kernel<<<blocks, 256, 0, stream>>>(x, r, rows, d, eps);
  return cudaGetLastError();
}

}  // namespace mom
