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

__device__ volatile int g_stop;
template <int KIND_F16, int TS, int SW>
__global__ void bench(int n, int iters, int pattern, unsigned long long* out, const float* gsrc = nullptr, int copy_kb = 0) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t cbar;
  __shared__ __align__(8) uint64_t ring[4];
  __shared__ volatile int done;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { done = 0; asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&cbar))); for (int r = 0; r < 4; ++r) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&ring[r]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
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
        if (pattern >= 4) acol += (it & 3) * 64;
        uint64_t bd = SW ? desc_sw128(b0 + boff) : desc_none(b0 + boff);
        uint64_t ad = SW ? desc_sw128(a0 + (q / 3) * 32) : desc_none(a0 + (q / 3) * 128 * 32);
        mma<KIND_F16, TS>(t + (it & 1) * 0, t + acol, ad, bd, id, (it | q) ? 1u : 0u);
      }
      if (pattern >= 2) {  // commit per chunk (as the engine's MMA thread does)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&ring[it & 3])));
      }
      if (pattern >= 3 && it >= 2) {  // wait for the commit of chunk it-2
        uint32_t ph = ((it - 2) >> 2) & 1;
        asm volatile("{.reg .pred p; W3: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W3;}" :: "r"(smem_u32(&ring[(it - 2) & 3])), "r"(ph));
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" :: "r"(smem_u32(&bar)));
    long long c1 = clock64();
    atomicAdd(out, (unsigned long long)(c1 - c0));
    done = 1;
  }
  if (threadIdx.x == 32 && copy_kb > 0) {
    uint32_t ph = 0; unsigned long long copies = 0;
    while (!done) {
      uint32_t bytes = copy_kb * 1024;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&cbar)), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(smem_u32(smem + 65536)), "l"(gsrc + (copies % 64) * 8192), "r"(bytes), "r"(smem_u32(&cbar)));
      asm volatile("{.reg .pred p; W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W2;}" :: "r"(smem_u32(&cbar)), "r"(ph));
      ph ^= 1; ++copies;
    }
    atomicAdd(out + 1, copies);
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}

template <int K, int T, int S>
void run(const char* name, int n, int pattern, int ctas, int copy_kb = 0) {
  unsigned long long* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
  static float* g = nullptr; if (!g) { cudaMalloc(&g, 64 * 8192 * 4 + 65536); cudaMemset(g, 0, 64 * 8192 * 4 + 65536); }
  cudaFuncSetAttribute(bench<K, T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  int iters = 200;
  bench<K, T, S><<<ctas, 128, 140000>>>(n, 10, pattern, d, g, copy_kb); cudaDeviceSynchronize(); cudaMemset(d, 0, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<K, T, S><<<ctas, 128, 140000>>>(n, iters, pattern, d, g, copy_kb);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long hh[2]; cudaMemcpy(hh, d, 16, cudaMemcpyDeviceToHost); unsigned long long h = hh[0];
  double cyc = (double)h / ctas / (iters * 12.0);
  double kdim = K ? 16 : 8;
  double tflops = 2.0 * 128 * n * kdim * iters * 12.0 * ctas / (ms * 1e-3) / 1e12;
  double cyc_total = (double)h / ctas;
  double copy_bpc = copy_kb ? (double)hh[1] * copy_kb * 1024 / ctas / cyc_total : 0;
  printf("%-34s N=%3d pattern=%d ctas=%3d copy=%2dKB : %7.1f cyc/MMA  (%.0f TFLOP/s chip) copy %.1f B/clk/SM err=%s\n", name, n, pattern, ctas, copy_kb, cyc, tflops, copy_bpc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int n : {16, 32, 48, 64, 80, 96, 112, 128, 144, 160, 192, 224, 256})
    run<0, 1, 0>("tf32 TS  B:none", n, 0, 148, 0);
  for (int n : {64, 96, 112, 128})
    run<0, 1, 0>("tf32 TS  B:none hi/lo+commit+wait", n, 3, 148, 0);
  return 0;
}
