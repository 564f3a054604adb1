// mlp_tc.cu -- tcgen05/TMEM/TMA kernels for the bf16 mini-sequence SwiGLU MLP
// (Alg. 1 P:109-113 of arXiv 2504.12526; MLP = SwiGLU).
//
// One persistent, warp-specialised "dual-B" GEMM kernel computes both phases of a mini-sequence:
//
//   Phase A  (gate/up + SiLU*mul):  acc[:, 0:128]   = X_i Wg[n0:n0+128]^T
//                                   acc[:, 128:256] = X_i Wu[n0:n0+128]^T
//            epilogue  H_i[:, n0:n0+128] = bf16( silu(acc[:, j]) * acc[:, 128+j] )
//   Phase B  (down + residual):     acc[:, 0:256]   = H_i Wd[n0:n0+256]^T
//            epilogue  out[:, n0:n0+256] = bf16( residual + acc )
//
// so one UMMA with N = 256 computes the gate and up tiles of the same 128 intermediate
// columns side by side in TMEM, and the [S, I] gate/up tensors never exist (Eq. 1).
//
// MODE_A / MODE_B run one phase per launch.  MODE_FUSED runs the whole mini-sequence in ONE
// persistent launch: tiles are ordered by groups of `group_m` 256-row blocks, each group's
// phase-A tiles followed by its phase-B tiles, and a phase-B tile's producer waits (acquire
// spin on a per-row-block counter that phase-A epilogues release) until all phase-A tiles of
// its row block have written H.  Phase B of group g thus overlaps phase A of group g+1: no
// launch gap and no wave-quantisation tail between the phases, and H rows are re-read soon
// after they were written.  Deadlock-free: a tile only waits on tiles with smaller indices,
// every CTA walks its tiles in increasing order, and the grid is co-resident (persistent).
//
// Roles (256 threads): warp 0 = TMA producer (1 lane), warp 1 = TMEM allocator + MMA issuer
// (1 lane), warps 4..7 = epilogue (TMEM lane quarter q = warp - 4, one row per thread).
// Pipelines: smem stages full/empty (TMA <-> MMA), TMEM accumulators full/empty x2
// (MMA <-> epilogue, 2 x 256 fp32 columns = all 512 TMEM columns).
//
// CG = 1: one CTA per tile, UMMA M = 128, the CTA stages both B halves (Wg and Wu rows).
// CG = 2: a CTA pair (cluster of 2) per tile, UMMA M = 256 (cta_group::2): CTA r stages
//         A rows [128r, 128r+128) and B half r; the leader CTA issues the MMAs; both CTAs
//         hold their 128 rows x 256 columns of the accumulator in their own TMEM.
//
// Determinism: no split-K, no atomics on data, the tile shape does not depend on the
// mini-sequence length, and every accumulator sums K in the same order -> outputs are bitwise
// identical for every mini-sequence count M and for fused vs unfused ("identical logits").
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "ptx.cuh"

namespace mom {

namespace tc {

constexpr uint32_t BM = 128;         // rows per CTA
constexpr uint32_t BK = 64;          // K per stage (64 bf16 = 128 B = one swizzle span)
constexpr uint32_t BHALF = 128;      // rows per B half
constexpr uint32_t UMMA_N = 256;     // both B halves
constexpr uint32_t UMMA_K = 16;      // fixed for kind::f16
constexpr uint32_t A_BYTES = BM * BK * 2;        // 16 KB
constexpr uint32_t BHALF_BYTES = BHALF * BK * 2; // 16 KB
constexpr uint32_t ACC_COLS = 256;
constexpr uint32_t NUM_THREADS = 256;
constexpr uint32_t EPI_WARP0 = 4;

enum : int { MODE_A = 0, MODE_B = 1, MODE_FUSED = 2 };

template <int CG>
struct Cfg {
  static constexpr uint32_t B_BYTES = (CG == 1 ? 2 : 1) * BHALF_BYTES;  // B bytes staged per CTA
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t STAGES = CG == 1 ? 4 : 6;
  static constexpr uint32_t TX_BYTES = STAGE_BYTES * CG;  // bytes landing per stage per tile
  static constexpr uint32_t EPI_STAGE_BYTES = 4 * 32 * 128;  // phase-B epilogue: 32 rows x 128 B per warp
  static constexpr uint32_t SMEM_BYTES =
      1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers*/ + EPI_STAGE_BYTES;
};

// The five operands of one mini-sequence (unused ones are copies in single-phase modes).
struct Maps {
  CUtensorMap x;   // A of phase A: X_i [C_i, d]
  CUtensorMap wg;  // B half 0 of phase A: W_gate [I, d]
  CUtensorMap wu;  // B half 1 of phase A: W_up [I, d]
  CUtensorMap h;   // A of phase B: H_i [C_i, I]
  CUtensorMap wd;  // B halves of phase B: W_down [d, I]
  CUtensorMap wg_h, wu_h;  // phase A half-width tail tiles: W_gate / W_up, 64-row boxes
};

struct Params {
  uint32_t rows;         // valid rows of this mini-sequence (C_i)
  uint32_t d, I;         // hidden, intermediate
  uint32_t m_tiles;      // ceil(rows / (BM*CG))
  uint32_t nA, nB;       // N tiles of phase A (I/128) and phase B (d/nb)
  uint32_t nb;           // phase-B tile width (UMMA N, multiple of 32, <= 256), chosen for wave quantisation
  uint32_t group_m;      // raster: row blocks per group (N iterates inside a group)
  uint32_t group_n;      // phase B only, if > 0: column-block groups instead (M iterates inside a group)
  uint32_t policy;       // TMA L2 policy: 0 reuse-aware (default), 1 all evict_normal, 2 A evict_first
  // Phase-A wave-tail split (MODE_A): tiles [0, n_full) are the usual 128-column tiles; the R tiles
  // that would form the last, partial wave are instead 2R half-width (64-column) tiles, so the last
  // wave takes half a tile time on up to 2R clusters (2R <= clusters).  n_half = 2R (0 = off).
  uint32_t n_full, n_half;
  __nv_bfloat16 *h;              // phase A output H_i [rows, I]
  __nv_bfloat16 *out;            // phase B output rows [rows, d]
  const __nv_bfloat16 *residual; // phase B residual, may be null
  const float *row_scale;        // phase A: folded-RMSNorm 1/rms per row, or null
  uint32_t *ready;               // MODE_FUSED: per (row block, CTA rank) count of finished phase-A tiles
  uint32_t coalesced_a;          // phase-A epilogue through the smem stage (128-B row segments)
  uint32_t fast_silu;            // phase-A epilogue: quotient of the SiLU by rcp.approx (no branch)
  unsigned long long *trace;     // instrumentation (mom_set_kernel_trace): 8 stamps per CTA, or null
  // L2 hints for the epilogues' streamed traffic (MOM_EPI_L2_HINT): bit 0 = phase-A H stores
  // evict_first (H is re-read only by the next launch, and displaces X_i rows that this launch
  // re-reads), bit 1 = phase-B residual loads and output stores evict_first
  uint32_t epi_hint;
  uint32_t n_peers;              // f1: extra destinations of the phase-B output rows
  __nv_bfloat16 *peer_out[kMaxPeers];  // f1: peers' gathered buffers, offset like `out`
  // f1 forwarding (warps 2-3): rows [0, fwd_rows) of fwd_src (the previous mini-sequence's
  // finished output) are copied to fwd_dst[0..n_fwd) during this launch
  const __nv_bfloat16 *fwd_src;
  uint32_t fwd_rows, n_fwd;
  __nv_bfloat16 *fwd_dst[kMaxPeers];
};

struct Tile {
  uint32_t m, n;
  bool a;       // phase A tile
  uint32_t c0;  // phase A: first H column (= first W_gate/W_up row) of the tile
  uint32_t hw;  // phase A: H columns of the tile (BHALF, or BHALF / 2 for a tail half tile)
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <int MODE>
__device__ __forceinline__ Tile decode_tile(uint32_t t, const Params &p) {
  Tile tl;
  uint32_t half = 0;
  bool is_half = false;
  if (MODE == MODE_A && t >= p.n_full) {  // tail half tile: the same raster slot as full tile n_full + h/2
    const uint32_t h = t - p.n_full;
    t = p.n_full + h / 2;
    half = h & 1u;
    is_half = true;
  }
  const uint32_t G = p.group_m;
  if constexpr (MODE == MODE_FUSED) {
    // Lagged order A0, (A1, B0), (A2, B1), ..., (A_{ng-1}, B_{ng-2}), B_{ng-1}: the phase-B tiles
    // of group g follow the phase-A tiles of group g+1, so by the time a CTA reaches them the
    // phase-A tiles they depend on finished long ago (no bubble at group boundaries).
    // Groups hold G row blocks except the last (rem = m_tiles % G); G <= m_tiles.
    const uint32_t full = p.m_tiles / G, rem = p.m_tiles % G;
    const uint32_t sA = G * p.nA, sB = G * p.nB;
    uint32_t g, gm, local;
    bool a;
    if (t < sA) {
      g = 0; gm = G; local = t; a = true;                          // A0
    } else {
      t -= sA;
      const uint32_t P = sA + sB;
      const uint32_t k = t / P;
      if (k + 1 < full) {                                          // regular pair (A_{k+1}, B_k)
        local = t - k * P;
        a = local < sA;
        g = a ? k + 1 : k;
        if (!a) local -= sA;
        gm = G;
      } else {
        t -= (full - 1) * P;
        if (rem > 0 && t < rem * p.nA) {                           // A_full (partial)
          g = full; gm = rem; local = t; a = true;
        } else {
          if (rem > 0) t -= rem * p.nA;
          if (t < sB) {                                            // B_{full-1}
            g = full - 1; gm = G; local = t; a = false;
          } else {                                                 // B_full (partial)
            g = full; gm = rem; local = t - sB; a = false;
          }
        }
      }
    }
    tl.a = a;
    tl.m = g * G + local % gm;
    tl.n = local / gm;
  } else if (MODE == MODE_B && p.group_n > 0) {
    // column-block groups: GN output-column panels of W_down stay hot while all row blocks of H_i
    // stream past them (tools/l2_model_phase_b.py: ~10 % fewer DRAM reads at GN = 8)
    const uint32_t GN = p.group_n;
    const uint32_t per_group = GN * p.m_tiles;
    const uint32_t g = t / per_group;
    const uint32_t local = t - g * per_group;
    const uint32_t n0 = g * GN;
    uint32_t gn = p.nB - n0;
    if (gn > GN) gn = GN;
    tl.n = n0 + local % gn;
    tl.m = local / gn;
    tl.a = false;
  } else {
    const uint32_t nt = MODE == MODE_A ? p.nA : p.nB;
    const uint32_t per_group = G * nt;
    const uint32_t g = t / per_group;
    const uint32_t local = t - g * per_group;
    const uint32_t m0 = g * G;
    uint32_t gm = p.m_tiles - m0;
    if (gm > G) gm = G;
    tl.m = m0 + local % gm;
    tl.n = local / gm;
    tl.a = MODE == MODE_A;
  }
  tl.hw = is_half ? BHALF / 2 : BHALF;
  tl.c0 = tl.n * BHALF + half * (BHALF / 2);
  return tl;
}

template <int MODE>
__host__ __device__ __forceinline__ uint32_t num_tiles_of(const Params &p) {
  return MODE == MODE_A ? (p.n_half ? p.n_full + p.n_half : p.m_tiles * p.nA)
                        : MODE == MODE_B ? p.m_tiles * p.nB : p.m_tiles * (p.nA + p.nB);
}

// Swish(g) * u = g * sigmoid(g) * u, fp32.  FAST: the quotient by rcp.approx (<= 2 ulp,
// no slow-path branch) instead of IEEE division, whose per-element FCHK/branch region kept the
// compiler from interleaving elements (the phase-A epilogue was latency-bound on it).
template <bool FAST>
__device__ __forceinline__ float silu_mul(float g, float u) {
  if constexpr (FAST) return __fdividef(g, 1.0f + __expf(-g)) * u;
  return g / (1.0f + __expf(-g)) * u;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Phase A epilogue for one tile: H[row, col0 + j] = bf16(silu(g_j * rs) * (u_j * rs)), j < 128.
// hw = H columns of the tile (gate accumulators at TMEM columns [0, hw), up at [hw, 2 hw)).
template <bool FAST>
__device__ __forceinline__ void epilogue_a(const Params &p, uint32_t taddr, uint32_t row, bool row_ok, uint32_t col0,
                                           uint32_t hw) {
  __nv_bfloat16 *orow = p.h + static_cast<size_t>(row) * p.I + col0;
  // folded RMSNorm (f3): gate/up of row r are scaled by r's 1/rms before the SiLU
  const float rs = (p.row_scale != nullptr && row_ok) ? p.row_scale[row] : 1.0f;
#pragma unroll 1
  for (uint32_t c = 0; c < hw / 32; ++c) {
    uint32_t g[32], u[32];
    ptx::tmem_ld_32x32b_x32(taddr + c * 32, g);
    ptx::tmem_ld_32x32b_x32(taddr + hw + c * 32, u);
    ptx::tmem_ld_wait();
    if (p.row_scale != nullptr) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        g[i] = __float_as_uint(__uint_as_float(g[i]) * rs);
        u[i] = __float_as_uint(__uint_as_float(u[i]) * rs);
      }
    }
    uint32_t packed[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float h0 = silu_mul<FAST>(__uint_as_float(g[2 * i]), __uint_as_float(u[2 * i]));
      float h1 = silu_mul<FAST>(__uint_as_float(g[2 * i + 1]), __uint_as_float(u[2 * i + 1]));
      packed[i] = ptx::pack_bf16x2(h0, h1);
    }
    if (row_ok) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        if (col0 + c * 32 + v * 8 < p.I) {
          uint4 w = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
          *reinterpret_cast<uint4 *>(orow + c * 32 + v * 8) = w;
        }
      }
    }
  }
}

// Phase A epilogue, coalesced variant: 64 H columns (128 B per row) at a time through the same
// per-warp 32 x 128 B XOR-swizzled stage as phase B, stored as full 128-B row segments.
template <bool FAST>
__device__ __forceinline__ void epilogue_a_coalesced(const Params &p, uint32_t taddr, uint32_t row0_warp,
                                                     uint32_t col0, uint32_t hw, uint8_t *stage) {
  const uint32_t lane = ptx::lane_id();
  const uint32_t row = row0_warp + lane;
  const uint32_t sbase = ptx::smem_u32(stage);
  auto sw = [&](uint32_t r, uint32_t v) { return sbase + r * 128 + (((v ^ r) & 7) << 4); };
  const uint32_t cr = lane >> 3, cv = lane & 7;
  const float rs = (p.row_scale != nullptr && row < p.rows) ? p.row_scale[row] : 1.0f;
#pragma unroll 1
  for (uint32_t c = 0; c < hw / 64; ++c) {
#pragma unroll
    for (uint32_t half = 0; half < 2; ++half) {  // 32 columns of g and u at a time (register budget)
      uint32_t g[32], u[32];
      ptx::tmem_ld_32x32b_x32(taddr + c * 64 + half * 32, g);
      ptx::tmem_ld_32x32b_x32(taddr + hw + c * 64 + half * 32, u);
      ptx::tmem_ld_wait();
#pragma unroll
      for (uint32_t v = 0; v < 4; ++v) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float g0 = __uint_as_float(g[8 * v + 2 * e]), g1 = __uint_as_float(g[8 * v + 2 * e + 1]);
          float u0 = __uint_as_float(u[8 * v + 2 * e]), u1 = __uint_as_float(u[8 * v + 2 * e + 1]);
          if (p.row_scale != nullptr) {
            g0 *= rs; g1 *= rs; u0 *= rs; u1 *= rs;
          }
          w[e] = ptx::pack_bf16x2(silu_mul<FAST>(g0, u0), silu_mul<FAST>(g1, u1));
        }
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sw(lane, half * 4 + v)), "r"(w[0]), "r"(w[1]),
                     "r"(w[2]), "r"(w[3])
                     : "memory");
      }
    }
    __syncwarp();
    const uint32_t ccol = col0 + c * 64;
#pragma unroll
    for (uint32_t i = 0; i < 8; ++i) {
      const uint32_t r = cr + 4 * i, grow = row0_warp + r, gcol = ccol + cv * 8;
      uint4 v;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "r"(sw(r, cv))
                   : "memory");
      if (grow < p.rows && gcol < p.I) {
        if (p.epi_hint & 1u)
          ptx::st_global_v4_hint(p.h + size_t(grow) * p.I + gcol, v, ptx::policy_evict_first());
        else
          *reinterpret_cast<uint4 *>(p.h + size_t(grow) * p.I + gcol) = v;
      }
    }
    __syncwarp();
  }
}

// Phase B epilogue for one tile: out[row, col0 + j] = bf16(residual + acc_j), j < 256, for the
// 32 rows of this warp (TMEM lane quarter q), 64 columns (128 B per row) at a time.  Rows live
// one per thread in TMEM, so the residual and the output go through a per-warp 32 x 128 B
// shared-memory stage (16-B units XOR-swizzled by row: conflict-free both ways) and are moved
// to/from global memory coalesced, 4 full 128-B row segments per warp instruction.  Every
// output chunk is stored to `out` and to each peer's gathered buffer (f1: the all-gather of
// token-sharded runs fused into this epilogue; peers are NVLink-mapped device pointers).
__device__ __forceinline__ void epilogue_b(const Params &p, uint32_t taddr, uint32_t row0_warp, uint32_t col0,
                                           uint8_t *stage) {
  const uint32_t lane = ptx::lane_id();
  const uint32_t sbase = ptx::smem_u32(stage);
  // 16-B unit v of row r of the stage lives at byte r*128 + ((v ^ r) & 7) * 16
  auto sw = [&](uint32_t r, uint32_t v) { return sbase + r * 128 + (((v ^ r) & 7) << 4); };
  const uint32_t cr = lane >> 3, cv = lane & 7;  // coalesced mapping: lane -> (row cr + 4i, unit cv)
  const uint32_t cend = col0 + p.nb < p.d ? col0 + p.nb : p.d;  // end of this tile's valid columns
#pragma unroll 1
  for (uint32_t c = 0; c < (p.nb + 63) / 64; ++c) {
    const uint32_t ccol = col0 + c * 64;  // first column of this chunk
    uint32_t a[64];
    ptx::tmem_ld_32x32b_x32(taddr + c * 64, *reinterpret_cast<uint32_t(*)[32]>(a));
    ptx::tmem_ld_32x32b_x32(taddr + c * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(a + 32));
    // residual chunk -> stage (coalesced global reads)
    if (p.residual) {
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i) {
        const uint32_t r = cr + 4 * i, grow = row0_warp + r, gcol = ccol + cv * 8;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (grow < p.rows && gcol < cend) {
          const __nv_bfloat16 *src = p.residual + size_t(grow) * p.d + gcol;
          v = (p.epi_hint & 2u) ? ptx::ld_global_v4_hint(src, ptx::policy_evict_first())
                                : *reinterpret_cast<const uint4 *>(src);
        }
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sw(r, cv)), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w)
                     : "memory");
      }
      __syncwarp();
    }
    ptx::tmem_ld_wait();
    // this thread's row: add residual in fp32, one RNE rounding, back into the stage
#pragma unroll
    for (uint32_t v = 0; v < 8; ++v) {
      float r[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (p.residual) {
        uint4 q;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                     : "r"(sw(lane, v))
                     : "memory");
        const __nv_bfloat162 *q2 = reinterpret_cast<const __nv_bfloat162 *>(&q);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(q2[e]);
          r[2 * e] = f.x;
          r[2 * e + 1] = f.y;
        }
      }
      const uint32_t w0 = ptx::pack_bf16x2(r[0] + __uint_as_float(a[8 * v + 0]), r[1] + __uint_as_float(a[8 * v + 1]));
      const uint32_t w1 = ptx::pack_bf16x2(r[2] + __uint_as_float(a[8 * v + 2]), r[3] + __uint_as_float(a[8 * v + 3]));
      const uint32_t w2 = ptx::pack_bf16x2(r[4] + __uint_as_float(a[8 * v + 4]), r[5] + __uint_as_float(a[8 * v + 5]));
      const uint32_t w3 = ptx::pack_bf16x2(r[6] + __uint_as_float(a[8 * v + 6]), r[7] + __uint_as_float(a[8 * v + 7]));
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sw(lane, v)), "r"(w0), "r"(w1), "r"(w2), "r"(w3)
                   : "memory");
    }
    __syncwarp();
    // stage -> out (+ peers), coalesced: 4 rows x 128 B per warp instruction
#pragma unroll
    for (uint32_t i = 0; i < 8; ++i) {
      const uint32_t r = cr + 4 * i, grow = row0_warp + r, gcol = ccol + cv * 8;
      uint4 v;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "r"(sw(r, cv))
                   : "memory");
      if (grow < p.rows && gcol < cend) {
        const size_t off = size_t(grow) * p.d + gcol;
        if (p.epi_hint & 2u)
          ptx::st_global_v4_hint(p.out + off, v, ptx::policy_evict_first());
        else
          *reinterpret_cast<uint4 *>(p.out + off) = v;
        for (uint32_t k = 0; k < p.n_peers; ++k) *reinterpret_cast<uint4 *>(p.peer_out[k] + off) = v;
      }
    }
    __syncwarp();
  }
}

template <int CG, int MODE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    mlp_tc_kernel(const __grid_constant__ Maps maps, const Params p) {
  using C = Cfg<CG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the SWIZZLE_128B atoms
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *smem_a = smem;                                   // STAGES x A_BYTES
  uint8_t *smem_b = smem + C::STAGES * A_BYTES;             // STAGES x B_BYTES
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *full = bars;                       // [STAGES]
  uint64_t *empty = bars + C::STAGES;          // [STAGES]
  uint64_t *tfull = bars + 2 * C::STAGES;      // [2]
  uint64_t *tempty = bars + 2 * C::STAGES + 2; // [2]
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * C::STAGES + 4);
  uint8_t *epi_stage = smem + C::STAGES * C::STAGE_BYTES + 256;  // phase-B epilogue staging, 4 x 4 KB

  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 8 + 0] = globaltimer_ns();  // entry
  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const uint32_t rank = (CG == 2) ? ptx::cluster_ctarank() : 0;
  const bool leader = (rank == 0);
  const uint32_t cluster_id = blockIdx.x / CG;
  const uint32_t num_clusters = gridDim.x / CG;
  const uint32_t num_tiles = num_tiles_of<MODE>(p);
  const uint32_t kbA = (p.d + BK - 1) / BK;  // phase A reduces over hidden
  const uint32_t kbB = (p.I + BK - 1) / BK;  // phase B reduces over intermediate

  if (warp == 0 && lane == 0) {
    if (MODE != MODE_B) {
      ptx::prefetch_tmap(&maps.x);
      ptx::prefetch_tmap(&maps.wg);
      ptx::prefetch_tmap(&maps.wu);
    }
    if (MODE != MODE_A) {
      ptx::prefetch_tmap(&maps.h);
      ptx::prefetch_tmap(&maps.wd);
    }
    for (uint32_t s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (uint32_t a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 4 * CG);  // one arrival per epilogue warp of every CTA
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc<CG>(tmem_holder, 2 * ACC_COLS);
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // PDL (split mode): let the next launch in the stream start as soon as SMs free up; its CTAs
  // run their prologue and whatever does not depend on this launch, then griddepcontrol.wait.
  // Both are no-ops when the launches carry no programmatic-serialization attribute.
  if (MODE != MODE_FUSED) pdl_launch_dependents();

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      // L2 policies: phase A re-reads X rows across all N tiles of a group (keep), streams W;
      // phase B keeps W_down (re-read by every row block), streams H.
      const uint64_t pol_keep = ptx::policy_evict_last();
      const uint64_t pol_norm = ptx::policy_evict_normal();
      const uint64_t pol_first = ptx::policy_evict_first();
      const uint32_t full_leader0 = (CG == 2) ? ptx::mapa(ptx::smem_u32(&full[0]), 0) : ptx::smem_u32(&full[0]);
      // phase B reads H_i, written by the preceding phase-A launch: wait for it (and, through its
      // own epilogue wait, for everything before it).  Phase A reads only X_i and the weights.
      if (MODE == MODE_B) pdl_wait();
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = cluster_id; t < num_tiles; t += num_clusters) {
        const Tile tl = decode_tile<MODE>(t, p);
        if (MODE == MODE_FUSED && !tl.a) {
          // H rows of this CTA's 128-row block must be complete: wait for every phase-A tile
          // of the block (released by their epilogues), then order the async-proxy (TMA) reads
          // after that acquire.
          const uint32_t *cnt = p.ready + tl.m * CG + rank;
          while (ld_acquire_gpu(cnt) < p.nA) __nanosleep(128);
          fence_proxy_async_global();
        }
        const bool half_a = tl.a && tl.hw < BHALF;
        const CUtensorMap *ta = tl.a ? &maps.x : &maps.h;
        const CUtensorMap *tb0 = tl.a ? (half_a ? &maps.wg_h : &maps.wg) : &maps.wd;
        const CUtensorMap *tb1 = tl.a ? (half_a ? &maps.wu_h : &maps.wu) : &maps.wd;
        uint64_t pol_a, pol_b;
        switch (p.policy) {
          case 1: pol_a = pol_norm; pol_b = pol_norm; break;                          // all normal
          case 2: pol_a = pol_first; pol_b = tl.a ? pol_norm : pol_keep; break;      // A streamed
          case 3: pol_a = tl.a ? pol_keep : pol_norm; pol_b = pol_first; break;      // weights streamed
          case 4: pol_a = pol_keep; pol_b = pol_first; break;                        // A kept, W streamed
          case 5: pol_a = tl.a ? pol_keep : pol_first; pol_b = tl.a ? pol_norm : pol_keep; break;  // H streamed
          default: pol_a = tl.a ? pol_keep : pol_norm; pol_b = tl.a ? pol_norm : pol_keep; break;
        }
        const int32_t a_row = static_cast<int32_t>(tl.m * BM * CG + rank * BM);
        const int32_t b_row0 = static_cast<int32_t>(tl.a ? tl.c0 : tl.n * p.nb);
        const int32_t b_off1 = tl.a ? 0 : static_cast<int32_t>(p.nb / 2);  // row offset of B half 1
        // bytes landing per stage: phase B's B halves are nb/2 rows (nb < 256 for some shapes)
        const uint32_t bhalf_bytes = tl.a ? tl.hw * BK * 2 : (p.nb / 2) * BK * 2;
        const uint32_t tx_bytes = (A_BYTES + (CG == 1 ? 2 : 1) * bhalf_bytes) * CG;
        const uint32_t num_kb = tl.a ? kbA : kbB;
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          const int32_t kc = static_cast<int32_t>(kb * BK);
          const uint32_t sa = ptx::smem_u32(smem_a + stage * A_BYTES);
          const uint32_t sb = ptx::smem_u32(smem_b + stage * C::B_BYTES);
          const uint32_t fbar = full_leader0 + stage * 8;
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], tx_bytes);
          if constexpr (CG == 1) {
            ptx::tma_load_2d(ta, sa, fbar, kc, a_row, pol_a);
            ptx::tma_load_2d(tb0, sb, fbar, kc, b_row0, pol_b);
            ptx::tma_load_2d(tb1, sb + bhalf_bytes, fbar, kc, b_row0 + b_off1, pol_b);
          } else {
            ptx::tma_load_2d_cg2(ta, sa, fbar, kc, a_row, pol_a);
            if (rank == 0)
              ptx::tma_load_2d_cg2(tb0, sb, fbar, kc, b_row0, pol_b);
            else
              ptx::tma_load_2d_cg2(tb1, sb, fbar, kc, b_row0 + b_off1, pol_b);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
      // Tail: wait until the MMA released every stage, so no tcgen05.commit arrival is still
      // in flight towards this CTA's shared memory when it exits.
      for (uint32_t i = 0; i < C::STAGES; ++i) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA, one thread) =======================
    if (leader && lane == 0) {
      constexpr uint32_t idesc_a = ptx::idesc_bf16_f32(BM * CG, UMMA_N);
      constexpr uint32_t idesc_a_half = ptx::idesc_bf16_f32(BM * CG, UMMA_N / 2);
      const uint32_t idesc_b = ptx::idesc_bf16_f32(BM * CG, p.nb);
      uint32_t stage = 0, phase = 0;
      uint32_t acc = 0, acc_phase = 0;
#ifdef MOM_TRACE_WAITS
      // probe build (-DMOM_TRACE_WAITS): MMA-issuer cycles spent waiting for operands (full) and for a
      // free accumulator (tempty), after the first stage of the launch; written to trace slots 6 / 7
      unsigned long long wait_full = 0, wait_acc = 0;
#endif
      for (uint32_t t = cluster_id; t < num_tiles; t += num_clusters) {
        const Tile tl = decode_tile<MODE>(t, p);
        const uint32_t num_kb = tl.a ? kbA : kbB;
        const uint32_t idesc = tl.a ? (tl.hw < BHALF ? idesc_a_half : idesc_a) : idesc_b;
#ifdef MOM_TRACE_WAITS
        const long long w0 = clock64();
#endif
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
#ifdef MOM_TRACE_WAITS
        if (p.trace && t != cluster_id) wait_acc += clock64() - w0;
#endif
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * ACC_COLS;
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
#ifdef MOM_TRACE_WAITS
          const long long w1 = clock64();
#endif
          ptx::mbar_wait(&full[stage], phase);
#ifdef MOM_TRACE_WAITS
          if (p.trace && (t != cluster_id || kb != 0)) wait_full += clock64() - w1;
#endif
          ptx::tc_fence_after();
          if (p.trace && kb == 0 && t == cluster_id) {  // first MMA: time and SM cycle counter
            p.trace[blockIdx.x * 8 + 1] = globaltimer_ns();
            p.trace[blockIdx.x * 8 + 4] = clock64();
          }
          const uint64_t adesc = ptx::sw128_kmajor_desc(ptx::smem_u32(smem_a + stage * A_BYTES));
          const uint64_t bdesc = ptx::sw128_kmajor_desc(ptx::smem_u32(smem_b + stage * C::B_BYTES));
#pragma unroll
          for (uint32_t k = 0; k < BK / UMMA_K; ++k) {
            // advance 16 bf16 = 32 B along K inside the 128-B swizzle span (>>4 -> +2)
            ptx::mma_bf16<CG>(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          ptx::mma_commit<CG>(&empty[stage], 0x3);  // frees the smem stage (both CTAs for CG=2)
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit<CG>(&tfull[acc], 0x3);      // accumulator ready for the epilogue(s)
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (p.trace) {  // last MMA issued
        p.trace[blockIdx.x * 8 + 2] = globaltimer_ns();
        p.trace[blockIdx.x * 8 + 5] = clock64();
#ifdef MOM_TRACE_WAITS
        p.trace[blockIdx.x * 8 + 6] = wait_full;
        p.trace[blockIdx.x * 8 + 7] = wait_acc;
#endif
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ======================= epilogue: TMEM -> registers -> global =======================
    const uint32_t q = warp - EPI_WARP0;  // TMEM lane quarter
    const uint32_t row_in_tile = q * 32 + lane;
    uint32_t acc = 0, acc_phase = 0;
    const uint32_t tempty_leader = (CG == 2) ? ptx::mapa(ptx::smem_u32(&tempty[0]), 0) : 0;
    // phase A writes H_i, which the preceding phase-B launch (previous mini-sequence) reads, and
    // reads row_scale; phase B writes O_i: no epilogue store before the previous launch completed
    pdl_wait();
    for (uint32_t t = cluster_id; t < num_tiles; t += num_clusters) {
      const Tile tl = decode_tile<MODE>(t, p);
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t row = tl.m * BM * CG + rank * BM + row_in_tile;
      const bool row_ok = row < p.rows;
      const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * ACC_COLS;
      const unsigned long long epi_t0 = p.trace ? clock64() : 0ull;
      if (tl.a && p.coalesced_a && p.fast_silu)
        epilogue_a_coalesced<true>(p, taddr, row - lane, tl.c0, tl.hw, epi_stage + q * 32 * 128);
      else if (tl.a && p.coalesced_a)
        epilogue_a_coalesced<false>(p, taddr, row - lane, tl.c0, tl.hw, epi_stage + q * 32 * 128);
      else if (tl.a && p.fast_silu)
        epilogue_a<true>(p, taddr, row, row_ok, tl.c0, tl.hw);
      else if (tl.a)
        epilogue_a<false>(p, taddr, row, row_ok, tl.c0, tl.hw);
      else
        epilogue_b(p, taddr, row - lane, tl.n * p.nb, epi_stage + q * 32 * 128);
#ifndef MOM_TRACE_WAITS
      if (p.trace && q == 0 && lane == 0) {  // epilogue cycles of warp 4 (summed) and tile count
        p.trace[blockIdx.x * 8 + 6] += clock64() - epi_t0;
        p.trace[blockIdx.x * 8 + 7] += 1;
      }
#endif
      // release the accumulator to the MMA issuer
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          ptx::mbar_arrive_cluster(tempty_leader + acc * 8);
        else
          ptx::mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (MODE == MODE_FUSED && tl.a) {
        // publish this tile's H rows: generic stores -> async proxy (TMA) of other CTAs
        fence_proxy_async_global();
        ptx::named_bar_sync(1, 128);  // all 4 epilogue warps of this CTA have stored
        if (q == 0 && lane == 0) {
          __threadfence();
          atomicAdd(p.ready + tl.m * CG + rank, 1u);
        }
      }
    }
  } else if (p.n_fwd > 0) {
    // ======================= warps 2-3: forward the previous mini-sequence's rows (f1) =========
    // Its output rows are final (the previous launch completed); copy this CTA's share of them
    // to every peer while the tensor cores work on this mini-sequence.  64 threads per CTA,
    // 16-B units, 4 independent loads in flight per thread.
    pdl_wait();  // the rows are final once the previous launch (its phase B) completed
    const uint32_t tid = threadIdx.x - 64;  // 0..63
    const size_t units = static_cast<size_t>(p.fwd_rows) * (p.d / 8);
    const size_t per_cta = (units + gridDim.x - 1) / gridDim.x;
    const size_t u0 = static_cast<size_t>(blockIdx.x) * per_cta;
    const size_t u1 = u0 + per_cta < units ? u0 + per_cta : units;
    const uint4 *src = reinterpret_cast<const uint4 *>(p.fwd_src);
    for (size_t u = u0 + tid; u < u1; u += 4 * 64) {
      uint4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (u + j * 64 < u1) v[j] = src[u + j * 64];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (u + j * 64 < u1)
          for (uint32_t k = 0; k < p.n_fwd; ++k) reinterpret_cast<uint4 *>(p.fwd_dst[k])[u + j * 64] = v[j];
    }
  }

  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, 2 * ACC_COLS);
  }
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 8 + 3] = globaltimer_ns();  // exit
}

template <int CG, int MODE>
static cudaError_t launch(const Maps &maps, const Params &p, int num_sms, bool pdl, cudaStream_t stream) {
  using C = Cfg<CG>;
  auto kfn = mlp_tc_kernel<CG, MODE>;
  static thread_local int configured_device = -1;  // attribute is per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (configured_device != dev) {
    e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured_device = dev;
  }
  const uint32_t num_tiles = num_tiles_of<MODE>(p);
  uint32_t clusters = static_cast<uint32_t>(num_sms) / CG;
  if (clusters > num_tiles) clusters = num_tiles;
  if (clusters == 0) clusters = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * CG, 1, 1);
  cfg.blockDim = dim3(NUM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  if (MODE == MODE_FUSED) {
    // phase-B tiles spin on counters released by phase-A tiles of OTHER clusters: every launched
    // cluster must be co-resident (MPS / green-context SM limits, cluster placement), so clamp the
    // grid to what can be active at once.  Tiles are taken in global order with a stride of the
    // cluster count, so any resident cluster count makes progress.
    int max_active = 0;
    e = cudaOccupancyMaxActiveClusters(&max_active, kfn, &cfg);
    if (e != cudaSuccess) return e;
    if (max_active < 1) return cudaErrorLaunchOutOfResources;
    if (clusters > static_cast<uint32_t>(max_active)) {
      clusters = static_cast<uint32_t>(max_active);
      cfg.gridDim = dim3(clusters * CG, 1, 1);
    }
  }
  return cudaLaunchKernelEx(&cfg, kfn, maps, p);
}

template <int MODE>
static cudaError_t launch_mode(const TcMlpArgs &a, cudaStream_t stream) {
  Maps maps;
  maps.x = *a.tm_x;
  maps.wg = *a.tm_wg;
  maps.wu = *a.tm_wu;
  maps.h = *a.tm_h;
  maps.wd = *a.tm_wd;
  maps.wg_h = a.tm_wg_h ? *a.tm_wg_h : *a.tm_wg;
  maps.wu_h = a.tm_wu_h ? *a.tm_wu_h : *a.tm_wu;
  Params p{};
  p.rows = a.rows;
  p.d = a.d;
  p.I = a.I;
  p.m_tiles = (a.rows + BM * a.cta_group - 1) / (BM * a.cta_group);
  p.nA = (a.I + BHALF - 1) / BHALF;
  p.nb = a.nb ? a.nb : UMMA_N;
  p.nB = (a.d + p.nb - 1) / p.nb;
  // raster groups (energy sweep r1): 16 row blocks for phase A (X rows stay in L2), 8 for B
  uint32_t g = a.group_m ? a.group_m : (MODE == MODE_B ? 8 : 16);
  if (g > p.m_tiles) g = p.m_tiles;
  p.group_m = g;
  p.group_n = MODE == MODE_B ? (a.group_n < p.nB ? a.group_n : p.nB) : 0;
  p.policy = a.policy;
  // phase-A wave tail: T tiles on `clusters` persistent clusters leave R = T mod clusters tiles for
  // a last partial wave; when 2R <= clusters they run as 2R half-width tiles (half a tile time)
  p.n_full = num_tiles_of<MODE>(p);
  p.n_half = 0;
  if (MODE == MODE_A && a.tm_wg_h && a.tm_wu_h) {
    const uint32_t T = p.m_tiles * p.nA;
    uint32_t clusters = static_cast<uint32_t>(a.num_sms) / a.cta_group;
    if (clusters > T) clusters = T;
    const uint32_t R = clusters ? T % clusters : 0;
    if (R > 0 && 2 * R <= clusters) {
      p.n_full = T - R;
      p.n_half = 2 * R;
    }
  }
  p.h = a.h;
  p.out = a.out;
  p.residual = a.residual;
  p.row_scale = a.row_scale;
  p.ready = a.ready;
  p.coalesced_a = a.coalesced_a;
  p.fast_silu = a.fast_silu;
  p.trace = a.trace;
  p.epi_hint = a.epi_hint;
  p.fwd_src = a.fwd_src;
  p.fwd_rows = a.fwd_rows;
  p.n_fwd = a.fwd_src ? a.n_fwd : 0;
  for (uint32_t k = 0; k < p.n_fwd && k < kMaxPeers; ++k) p.fwd_dst[k] = a.fwd_dst[k];
  p.n_peers = a.n_peers;
  for (uint32_t k = 0; k < a.n_peers && k < kMaxPeers; ++k) p.peer_out[k] = a.peer_out[k];
  const bool pdl = a.pdl && MODE != MODE_FUSED;
  if (a.cta_group == 2) return launch<2, MODE>(maps, p, a.num_sms, pdl, stream);
  return launch<1, MODE>(maps, p, a.num_sms, pdl, stream);
}

}  // namespace tc

cudaError_t launch_mlp_tc(const TcMlpArgs &a, int mode, cudaStream_t stream) {
  switch (mode) {
    case 0: return tc::launch_mode<tc::MODE_A>(a, stream);
    case 1: return tc::launch_mode<tc::MODE_B>(a, stream);
    default: return tc::launch_mode<tc::MODE_FUSED>(a, stream);
  }
}

size_t mlp_tc_ready_counters(uint32_t rows) { return (rows + tc::BM - 1) / tc::BM + 2; }

}  // namespace mom
