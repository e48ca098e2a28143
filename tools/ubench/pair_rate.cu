// Microbenchmark: cycles per kind::f16 tcgen05.mma, A from TMEM, B from SMEM
// (SWIZZLE_NONE K-major), single CTA (cta_group::1, M=128) vs CTA pair
// (cta_group::2, M=256, B split by N across the pair) -- is the pair MMA itself
// as fast per SM as the single-CTA one?  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pair_rate pair_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32; d |= (uint64_t)1 << 46; return d; }
__device__ __forceinline__ uint32_t idesc(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24); }

template <int PAIR>
__global__ void bench(int n, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)smem)[i] = 0.f;
  uint32_t crank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  if (threadIdx.x < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t t = slot;
  if (threadIdx.x == 0 && crank == 0) {
    const uint32_t b0 = smem_u32(smem);
    const uint32_t id = idesc(PAIR ? 256 : 128, n);
    const int nb = PAIR ? n / 2 : n;  // B rows held by this CTA
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int q = 0; q < 12; ++q) {
        const uint32_t acol = 416 + (q % 3 == 1 ? 8 : 0) + (it % 6) * 16 % 96;
        const uint32_t boff = ((q % 3 == 2) ? nb * 32 : 0) + (q / 3) * 2 * nb * 32;
        const uint64_t bd = desc_none(b0 + boff);
        const uint32_t d = t + ((it >> 1) & 1) * 208;
        const uint32_t acc = (it | q) ? 1u : 0u;
        if (PAIR)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;}" :: "r"(d), "r"(t + acol), "l"(bd), "r"(id), "r"(acc));
        else
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" :: "r"(d), "r"(t + acol), "l"(bd), "r"(id), "r"(acc));
      }
    }
    if (PAIR)
      asm volatile("{.reg .b16 m; mov.b16 m, 3; tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;}" :: "r"(smem_u32(&bar)));
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" :: "r"(smem_u32(&bar)));
    long long c1 = clock64();
    atomicAdd(out, (unsigned long long)(c1 - c0));
    atomicAdd(out + 1, 1ull);
  }
  if (PAIR && threadIdx.x == 0 && crank == 1)
    asm volatile("{.reg .pred p; W1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W1;}" :: "r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(t));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
  }
}

template <int PAIR>
void run(int n, int ctas) {
  unsigned long long* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
  auto fn = bench<PAIR>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  cudaLaunchConfig_t c{}; cudaLaunchAttribute at{};
  at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = PAIR ? 2 : 1; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
  c.gridDim = dim3(ctas); c.blockDim = dim3(128); c.dynamicSmemBytes = 140000; c.attrs = &at; c.numAttrs = 1;
  int iters = 10;
  cudaLaunchKernelEx(&c, fn, n, iters, d); cudaDeviceSynchronize(); cudaMemset(d, 0, 16);
  iters = 400;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&c, fn, n, iters, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double cyc = (double)h[0] / h[1] / (iters * 12.0);
  const double m = PAIR ? 256 : 128;
  const double tf = 2.0 * m * n * 16 * iters * 12.0 * h[1] / (ms * 1e-3) / 1e12;
  printf("%s N=%3d ctas=%3d issuers=%3llu : %7.1f cyc/MMA  (%.0f TFLOP/s chip, %.0f per-SM-equivalent cyc) err=%s\n",
         PAIR ? "pair  cta_group::2 M=256" : "single cta_group::1 M=128", n, ctas, h[1], cyc, tf,
         PAIR ? cyc : cyc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int n : {128, 208, 256}) { run<0>(n, 148); run<1>(n, 148); }
  return 0;
}
