// kernels.h -- internal launcher interface between the C ABI (api.cu) and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mom {

constexpr uint32_t kMaxTraceCtas = 160;  // mom_set_kernel_trace: 8 stamps per CTA per launch
constexpr uint32_t kMaxPeers = 7;  // f1: up to 8 GPUs (7 peers) receive every phase-B output row

// One mini-sequence on the tcgen05 path (mlp_tc.cu).  Tensor maps are 2D bf16, box 64 x 128.
struct TcMlpArgs {
  const CUtensorMap *tm_x;   // X_i [C_i, d]    (phase A operand A)
  const CUtensorMap *tm_wg;  // W_gate [I, d]   (phase A B half 0)
  const CUtensorMap *tm_wu;  // W_up [I, d]     (phase A B half 1)
  const CUtensorMap *tm_h;   // H_i [C_i, I]    (phase B operand A)
  const CUtensorMap *tm_wd;  // W_down [d, I]   (phase B B halves)
  const CUtensorMap *tm_wg_h;  // W_gate / W_up with a 64-row box: phase-A half-width tail tiles
  const CUtensorMap *tm_wu_h;  //   (null: no half tiles)
  uint32_t rows;             // C_i
  uint32_t d, I;
  __nv_bfloat16 *h;          // H_i (workspace)
  __nv_bfloat16 *out;        // out rows of this mini-sequence
  const __nv_bfloat16 *residual;  // may be null
  const float *row_scale;    // folded RMSNorm 1/rms per row (phase A), or null
  uint32_t *ready;           // fused mode: mlp_tc_ready_counters(rows) zeroed counters
  uint32_t coalesced_a;      // phase-A epilogue via the smem stage (coalesced H stores)
  uint32_t fast_silu;        // phase-A epilogue SiLU quotient by rcp.approx (MOM_FAST_SILU, default 1)
  unsigned long long *trace; // instrumentation: kMaxTraceCtas x 8 stamps for this launch, or null
  uint32_t epi_hint;         // MOM_EPI_L2_HINT: bit 0 H stores evict_first, bit 1 phase-B residual/out evict_first
  uint32_t n_peers;          // f1: number of peer destinations (<= kMaxPeers)
  __nv_bfloat16 *peer_out[kMaxPeers];  // f1: peer gathered buffers at this mini-sequence's rows
  const __nv_bfloat16 *fwd_src;        // f1: previous mini-sequence's output rows to forward (or null)
  uint32_t fwd_rows, n_fwd;            //     ... its row count and number of destinations
  __nv_bfloat16 *fwd_dst[kMaxPeers];   //     ... the peers' buffers at those rows
  uint32_t nb;               // phase-B tile width (multiple of 32, <= 256; 0 = 256); W_down map box = nb/2 rows
  int cta_group;             // 1 or 2
  uint32_t group_m;          // raster group (0 = default)
  uint32_t group_n;          // phase B column-group raster (0 = row groups)
  bool pdl;                  // launch with programmatic stream serialization (split mode)
  uint32_t policy;           // TMA L2 cache policy variant (0 = default)
  int num_sms;
};
// mode 0: phase A only, 1: phase B only, 2: both phases in one persistent launch.
cudaError_t launch_mlp_tc(const TcMlpArgs &a, int mode, cudaStream_t stream);
size_t mlp_tc_ready_counters(uint32_t rows);

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
// norm_eps >= 0: x is RMS-normalised first (f3; the gain folded into wg / wu by the caller)
cudaError_t launch_last_token_mlp(const void *x, const void *residual, const void *wg, const void *wu,
                                  const void *wd, void *out, float *h_ws, int d, int I, bool is_bf16,
                                  int num_sms, cudaStream_t stream, float norm_eps = -1.0f);
size_t lm_head_partials(int num_sms);
cudaError_t launch_lm_head(const void *h, const void *gain, float eps, const void *w, float *logits,
                           int32_t *argmax, unsigned long long *key_out, int vocab_offset,
                           unsigned long long *partials, int d, int V, bool is_bf16, int num_sms,
                           cudaStream_t stream);
cudaError_t launch_key_to_index(const unsigned long long *key, int32_t *argmax, cudaStream_t stream);

}  // namespace mom
