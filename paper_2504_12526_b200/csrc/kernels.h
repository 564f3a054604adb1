// kernels.h -- internal launcher interface between the C ABI (api.cu) and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mom {

// One phase of one mini-sequence on the tcgen05 path (mlp_tc.cu).
struct TcPhaseArgs {
  const CUtensorMap *tm_a;   // A operand rows (X_i for phase A, H_i for phase B), box 64 x 128
  const CUtensorMap *tm_b0;  // phase A: W_gate; phase B: W_down
  const CUtensorMap *tm_b1;  // phase A: W_up;   phase B: W_down (second 128-row half)
  uint32_t rows;             // C_i
  uint32_t n_out;            // I (phase A) or hidden (phase B)
  uint32_t k;                // hidden (phase A) or I (phase B)
  __nv_bfloat16 *out;        // H_i or out rows
  const __nv_bfloat16 *residual;  // phase B, may be null
  uint32_t ld_out;           // row pitch of out/residual in elements
  int cta_group;             // 1 or 2
  uint32_t group_m;          // raster group (0 = default)
  uint32_t policy;           // TMA L2 cache policy variant (0 = default)
  const float *row_scale;    // phase A only: per-row scale of the gate/up accumulators (folded RMSNorm), or null
  int num_sms;
};
cudaError_t launch_phase_a_tc(const TcPhaseArgs &a, cudaStream_t stream);
cudaError_t launch_phase_b_tc(const TcPhaseArgs &a, cudaStream_t stream);

// folded RMSNorm (norm.cu)
cudaError_t launch_fold_gain(const __nv_bfloat16 *w, const __nv_bfloat16 *g, __nv_bfloat16 *out, int64_t rows,
                             int64_t cols, int num_sms, cudaStream_t stream);
cudaError_t launch_row_inv_rms(const __nv_bfloat16 *x, float *r, int rows, int d, float eps, int num_sms,
                               cudaStream_t stream);

// fp32 SIMT path (mlp_simt.cu), row pointers already offset to the mini-sequence.
cudaError_t launch_phase_a_f32(const float *x, const float *wg, const float *wu, float *h, int rows, int d, int I,
                               cudaStream_t stream);
cudaError_t launch_phase_b_f32(const float *h, const float *wd, const float *residual, float *out, int rows, int d,
                               int I, cudaStream_t stream);

// GEMV path (gemv.cu).  is_bf16 selects bf16 vs fp32 storage of x/w/out.
cudaError_t launch_last_token_mlp(const void *x, const void *residual, const void *wg, const void *wu,
                                  const void *wd, void *out, float *h_ws, int d, int I, bool is_bf16,
                                  int num_sms, cudaStream_t stream);
size_t lm_head_partials(int num_sms);
cudaError_t launch_lm_head(const void *h, const void *gain, float eps, const void *w, float *logits,
                           int32_t *argmax, unsigned long long *key_out, int vocab_offset,
                           unsigned long long *partials, int d, int V, bool is_bf16, int num_sms,
                           cudaStream_t stream);
cudaError_t launch_key_to_index(const unsigned long long *key, int32_t *argmax, cudaStream_t stream);

}  // namespace mom
