// Minimal reproducer for the compute-sanitizer racecheck report on the TMEM-address hand-off
// (profiles/r1_sanitizer_racecheck.log: "Race ... Write access at mlp_tc_kernel+0x..fe80 and Read
// access at tmem_alloc ... ptx.cuh:127", cta_group::2 launches only).
// The pattern is the PTX-prescribed one: warp 1 runs tcgen05.alloc (the hardware writes the TMEM
// address to shared memory), tcgen05.fence::before_thread_sync, a barrier, tcgen05.fence::after_
// thread_sync, then every thread reads the address.  Variant 0 uses barrier.cluster arrive/wait as
// the barrier (what mlp_tc_kernel<2,*> does), variant 1 adds a __syncthreads() after it, variant 2
// is the one-CTA form (cta_group::1, __syncthreads only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tmem_rc tools/repro/tmem_alloc_racecheck.cu
// Run:   compute-sanitizer --tool racecheck /tmp/tmem_rc <variant>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int CG>
__global__ void alloc_kernel(unsigned *out, int variant) {
  __shared__ unsigned holder;
  const unsigned warp = threadIdx.x / 32;
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)),
                   "r"(256) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)),
                   "r"(256) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (variant == 1) __syncthreads();
  } else {
    __syncthreads();
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned taddr = holder;
  out[blockIdx.x * blockDim.x + threadIdx.x] = taddr;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(256) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(256) : "memory");
  }
}

int main(int argc, char **argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  const int blocks = 4, threads = 128;
  unsigned *out = nullptr;
  cudaMalloc(&out, blocks * threads * sizeof(unsigned));
  cudaError_t e;
  if (variant == 2) {
    alloc_kernel<1><<<blocks, threads>>>(out, variant);
    e = cudaGetLastError();
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, alloc_kernel<2>, out, variant);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  unsigned h[blocks * threads];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  bool same = true;  // every thread of a CTA read the same TMEM address
  for (int b = 0; b < blocks; ++b)
    for (int t = 1; t < threads; ++t) same &= h[b * threads + t] == h[b * threads];
  printf("variant %d: %s, consistent addresses: %s\n", variant, cudaGetErrorString(e), same ? "yes" : "no");
  return e == cudaSuccess && same ? 0 : 1;
}
