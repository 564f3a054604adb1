// Energy per byte of L2 -> shared-memory traffic: unicast bulk copies vs cluster multicast.
// Clusters of CS CTAs (one per SM) stream the same 32 KB blocks of a buffer that stays in L2 (48 MB):
//   unicast:   every CTA copies the whole block into its own shared memory (CS x the L2 reads)
//   multicast: CTA r copies 1/CS of the block and multicasts it to all CS CTAs of the cluster
// Every CTA receives the same bytes either way.  Host measures time and board energy (NVML) over
// >= 2 s per mode.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2mc l2_multicast_energy.cu -lnvidia-ml
#include <cuda_runtime.h>
#include <nvml.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <chrono>

constexpr int BLOCK = 32 * 1024;  // bytes per stage
constexpr int STAGES = 4;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}"
               ::"r"(smem_u32(b)), "r"(parity), "r"(0x989680) : "memory");
}

template <int CS, bool MC>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(128, 1) stream(const uint8_t *src, size_t nbytes, int iters, unsigned long long *sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[STAGES];
  const uint32_t rank = CS > 1 ? ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync();
  const size_t nblocks = nbytes / BLOCK;
  const size_t cluster = blockIdx.x / CS, nclusters = gridDim.x / CS;
  unsigned long long acc = 0;
  uint32_t phase[STAGES] = {0, 0, 0, 0};
  int it = 0;
  for (int rep = 0; rep < iters; ++rep) {
    for (size_t b0 = cluster * STAGES; b0 + STAGES <= nblocks; b0 += nclusters * STAGES) {
      if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
          expect_tx(&full[s], BLOCK);
          const uint8_t *g = src + (b0 + s) * BLOCK;
          const uint32_t dst = smem_u32(smem + s * BLOCK);
          if (MC) {
            const uint32_t part = BLOCK / CS;
            const uint16_t mask = (1u << CS) - 1;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                         ::"r"(dst + rank * part), "l"(g + rank * part), "r"(part), "r"(smem_u32(&full[s])), "h"(mask) : "memory");
          } else {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst), "l"(g), "r"(BLOCK), "r"(smem_u32(&full[s])) : "memory");
          }
        }
      }
      for (int s = 0; s < STAGES; ++s) mbar_wait(&full[s], phase[s]), phase[s] ^= 1;
      acc += smem[(threadIdx.x * 97 + it) % (STAGES * BLOCK)];
      ++it;
      // every CTA of the cluster must be done reading before anyone multicasts into the stages again
      cluster_sync();
    }
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

template <int CS, bool MC>
static void run(const char *name, const uint8_t *buf, size_t nbytes, int sms, nvmlDevice_t dev, unsigned long long *sink) {
  auto k = stream<CS, MC>;
  const int smem = STAGES * BLOCK;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = (sms / CS) * CS;
  k<<<grid, 128, smem>>>(buf, nbytes, 2, sink);  // warm-up
  cudaDeviceSynchronize();
  // calibrate iterations for ~2.5 s
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<grid, 128, smem>>>(buf, nbytes, 20, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  const int iters = static_cast<int>(20 * 2500.0 / ms) + 1;
  unsigned long long j0 = 0, j1 = 0;
  nvmlDeviceGetTotalEnergyConsumption(dev, &j0);
  cudaEventRecord(e0); k<<<grid, 128, smem>>>(buf, nbytes, iters, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
  nvmlDeviceGetTotalEnergyConsumption(dev, &j1);
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned int clk = 0; nvmlDeviceGetClockInfo(dev, NVML_CLOCK_SM, &clk);
  const double delivered = static_cast<double>(nbytes / (STAGES * BLOCK) * STAGES * BLOCK) * iters * (grid / CS) * CS / (grid / CS);
  // bytes landing in shared memory across all CTAs: each cluster covers its share of the buffer, every CTA gets it
  const double landed = static_cast<double>((nbytes / BLOCK) / STAGES * STAGES) * BLOCK * iters * CS;
  const double j = (j1 - j0) / 1e3;
  printf("{\"mode\": \"%s\", \"cs\": %d, \"ms\": %.1f, \"landed_GB\": %.1f, \"landed_TBps\": %.2f, \"J\": %.1f, \"W\": %.0f, \"pJ_per_landed_B\": %.2f, \"sm_mhz_end\": %u}\n",
         name, CS, ms, landed / 1e9, landed / (ms * 1e-3) / 1e12, j, j / (ms * 1e-3), j / landed * 1e12, clk);
  (void)delivered;
}

int main() {
  nvmlInit();
  nvmlDevice_t dev; nvmlDeviceGetHandleByIndex(0, &dev);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t nbytes = 48ull << 20;
  uint8_t *buf; cudaMalloc(&buf, nbytes); cudaMemset(buf, 1, nbytes);
  unsigned long long *sink; cudaMalloc(&sink, 8);
  for (int round = 0; round < 2; ++round) {
    run<4, false>("unicast", buf, nbytes, sms, dev, sink);
    run<4, true>("multicast", buf, nbytes, sms, dev, sink);
    run<2, false>("unicast", buf, nbytes, sms, dev, sink);
    run<2, true>("multicast", buf, nbytes, sms, dev, sink);
  }
  cudaError_t e = cudaGetLastError();
  printf("{\"cuda\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
