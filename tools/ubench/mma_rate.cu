// Microbenchmark: cycles per tcgen05.mma on this B200 for the patterns the
// ICNNM engine uses (kind::tf32, M=128, A from TMEM or SMEM, B from SMEM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32; d |= (uint64_t)1 << 46; return d; }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d; }
__device__ __forceinline__ uint32_t idesc(int kind_f16, int n) {
  uint32_t fmt = kind_f16 ? 1u : 2u;  // bf16 : tf32
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24); }

template <int KIND_F16, int TS>
__device__ __forceinline__ void mma(uint32_t d, uint32_t a_t, uint64_t a_d, uint64_t b, uint32_t id, uint32_t acc) {
  if (TS) {
    if (KIND_F16) asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" :: "r"(d), "r"(a_t), "l"(b), "r"(id), "r"(acc));
    else asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}" :: "r"(d), "r"(a_t), "l"(b), "r"(id), "r"(acc));
  } else {
    if (KIND_F16) asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" :: "r"(d), "l"(a_d), "l"(b), "r"(id), "r"(acc));
    else asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}" :: "r"(d), "l"(a_d), "l"(b), "r"(id), "r"(acc));
  }
}

template <int KIND_F16, int TS, int SW>
__global__ void bench(int n, int iters, int pattern, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t t = slot;
  if (threadIdx.x == 0) {
    uint32_t b0 = smem_u32(smem), a0 = smem_u32(smem + 32768);
    uint32_t id = idesc(KIND_F16, n);
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int q = 0; q < 12; ++q) {
        uint32_t acol = (pattern == 0) ? 256 : 256 + (q % 3 == 1 ? 32 : 0) + (q / 3) * 8;
        uint32_t boff = (pattern == 0) ? 0 : ((q % 3 == 2) ? 16384 : 0) + (SW ? (q / 3) * 32 : (q / 3) * n * 32);
        uint64_t bd = SW ? desc_sw128(b0 + boff) : desc_none(b0 + boff);
        uint64_t ad = SW ? desc_sw128(a0 + (q / 3) * 32) : desc_none(a0 + (q / 3) * 128 * 32);
        mma<KIND_F16, TS>(t + (it & 1) * 0, t + acol, ad, bd, id, (it | q) ? 1u : 0u);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" :: "r"(smem_u32(&bar)));
    long long c1 = clock64();
    atomicAdd(out, (unsigned long long)(c1 - c0));
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}

template <int K, int T, int S>
void run(const char* name, int n, int pattern, int ctas) {
  unsigned long long* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  cudaFuncSetAttribute(bench<K, T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  int iters = 200;
  bench<K, T, S><<<ctas, 128, 100000>>>(n, 10, pattern, d); cudaDeviceSynchronize(); cudaMemset(d, 0, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<K, T, S><<<ctas, 128, 100000>>>(n, iters, pattern, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  double cyc = (double)h / ctas / (iters * 12.0);
  double kdim = K ? 16 : 8;
  double tflops = 2.0 * 128 * n * kdim * iters * 12.0 * ctas / (ms * 1e-3) / 1e12;
  printf("%-34s N=%3d pattern=%d ctas=%3d : %7.1f cyc/MMA  (%.0f TFLOP/s chip)  err=%s\n", name, n, pattern, ctas, cyc, tflops, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int ctas : {1, 148}) {
    run<0, 1, 0>("tf32 TS  B:none", 128, 0, ctas);
    run<0, 1, 0>("tf32 TS  B:none (hi/lo pattern)", 128, 1, ctas);
    run<0, 1, 1>("tf32 TS  B:sw128 (hi/lo pattern)", 128, 1, ctas);
    run<0, 0, 0>("tf32 SS  A,B:none", 128, 0, ctas);
    run<0, 0, 1>("tf32 SS  A,B:sw128", 128, 0, ctas);
    run<0, 1, 0>("tf32 TS  B:none", 256, 0, ctas);
    run<0, 1, 0>("tf32 TS  B:none", 64, 0, ctas);
    run<1, 1, 0>("bf16 TS  B:none", 128, 0, ctas);
    run<1, 0, 1>("bf16 SS  A,B:sw128", 128, 0, ctas);
    run<1, 0, 1>("bf16 SS  A,B:sw128", 256, 0, ctas);
  }
  return 0;
}
