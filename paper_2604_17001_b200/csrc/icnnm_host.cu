// Host driver of the B200 ICNNM hot path: the C ABI of include/icnnm_b200.h.
//
// Mirrors the reference's C++ solver/operator API
// (/root/reference/proj/core/include/icnnm/{solver,conv_op,spectral}.hpp):
// validation rules and error classes follow solver.cpp:26-40,66-72,
// tensor.hpp:100-107,115-121 and spectral.cpp:25-41; the ADMM loop is the
// restated form of solver.cpp:62-146 documented in DESIGN.md §2.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <array>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/icnnm_b200.h"
#include "icnnm_comm.h"
#include "icnnm_kernels.cuh"
#include "icnnm_tc.cuh"

#include "icnnm_host_common.h"

using icnnm_dev::IterState;
using icnnm_dev::IterStats;

namespace icnnm_host {

thread_local std::string g_last_error;

#ifdef ICNNM_EXPERIMENTS
int env_knob(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
#endif

// ICNNM_TIMING=1: host-side phase times of the C-ABI calls on stderr (where an
// end-to-end call spends its time outside the device-resident loop).
struct PhaseTimer {
  bool on = std::getenv("ICNNM_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void reset() { t = std::chrono::steady_clock::now(); }
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[icnnm timing] %-24s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};
thread_local PhaseTimer g_timer;

// ---------------------------------------------------------------------------
// Device memory cache (declared in icnnm_host_common.h)
// ---------------------------------------------------------------------------
namespace {
struct CachedBlock {
  void* p;
  size_t bytes;
  int dev;
};
std::mutex g_cache_mu;
std::vector<CachedBlock> g_cache;
bool cache_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ICNNM_DEVCACHE");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}
void cache_flush_device(int dev) {  // caller holds g_cache_mu
  size_t w = 0;
  for (size_t i = 0; i < g_cache.size(); ++i) {
    if (g_cache[i].dev == dev)
      cudaFree(g_cache[i].p);
    else
      g_cache[w++] = g_cache[i];
  }
  g_cache.resize(w);
}
}  // namespace

void* devcache_alloc(size_t bytes) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (cache_enabled()) {
    // smallest cached block of this device that fits without wasting > 1/8
    size_t best = g_cache.size();
    for (size_t i = 0; i < g_cache.size(); ++i) {
      const CachedBlock& c = g_cache[i];
      if (c.dev == dev && c.bytes >= bytes && c.bytes - bytes <= c.bytes / 8 &&
          (best == g_cache.size() || c.bytes < g_cache[best].bytes))
        best = i;
    }
    if (best < g_cache.size()) {
      void* p = g_cache[best].p;
      g_cache.erase(g_cache.begin() + static_cast<std::ptrdiff_t>(best));
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();  // clear, hand the cached blocks back, retry once
    cache_flush_device(dev);
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(ICNNM_CUDA_ERROR,
         "cudaMalloc(" + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
  }
  return p;
}

void devcache_free(void* p, size_t bytes) {
  if (!p) return;
  if (!cache_enabled()) {
    cudaFree(p);
    return;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaFree(p);
    return;
  }
  // unwinding from an error: work on the block may still be in flight.  Solver
  // state is freed after ~Solver synchronised its own stream; the operator
  // entry points work on the legacy default stream.  (Not cudaDeviceSynchronize:
  // it would invalidate a stream capture running on another thread of a batch
  // call on the same device.)
  if (std::uncaught_exceptions() > 0) cudaStreamSynchronize(cudaStreamLegacy);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache.push_back({p, bytes, dev});
}

void devcache_empty() {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return;
  int prev = 0;
  cudaGetDevice(&prev);
  for (int d = 0; d < n; ++d) {
    bool any = false;
    for (auto& c : g_cache) any = any || c.dev == d;
    if (!any) continue;
    cudaSetDevice(d);
    cache_flush_device(d);
  }
  cudaSetDevice(prev);
}

// DenseTensor / KernelShape::validate_for (tensor.hpp:81-107).
Problem make_problem(int order, const int64_t* dims, const int64_t* kdims) {
  if (order < 1) invalid("DenseTensor: order must be >= 1");
  if (order > 3) invalid("icnnm_b200: tensor order > 3 is not supported");
  if (!dims || !kdims) invalid("null dims");
  Problem p;
  p.order = order;
  for (int j = 0; j < order; ++j) {
    if (dims[j] < 1) invalid("DenseTensor: dims must be positive");
    if (kdims[j] < 1 || kdims[j] > dims[j]) invalid("KernelShape: kernel dim out of range");
    p.dims[3 - order + j] = dims[j];
    p.kd[3 - order + j] = kdims[j];
  }
  p.m = p.dims[0] * p.dims[1] * p.dims[2];
  int64_t k = p.kd[0] * p.kd[1] * p.kd[2];
  if (p.dims[0] > (1 << 30) || p.m > (int64_t(1) << 40)) invalid("tensor too large");
  if (k > 4096) invalid("icnnm_b200: kernel with more than 4096 taps is not supported");
  p.k = static_cast<int>(k);
  p.kp = static_cast<int>(roundup(k, BN));
  p.kp_tc = static_cast<int>(roundup(k, icnnm_dev::tc::KC));
  return p;
}

// Launch geometry for `rows` H-rows of the tensor.  wrap=1: periodic over the
// whole tensor; wrap=0: slab buffer with kh-1 halo rows before the own rows.
Geo make_geo(const Problem& p, int64_t rows, bool wrap) {
  Geo g{};
  g.H = static_cast<int>(rows);
  g.W = static_cast<int>(p.dims[1]);
  g.T = static_cast<int>(p.dims[2]);
  g.kh = static_cast<int>(p.kd[0]);
  g.kw = static_cast<int>(p.kd[1]);
  g.kt = static_cast<int>(p.kd[2]);
  g.bt = g.T > 8 ? 16 : 8;
  const int rem = BM / g.bt;
  if (g.H == 1) {
    g.bh = 1;
    g.bw = rem;
  } else {
    g.bw = std::min(pow2ceil(g.W), 4);
    g.bh = rem / g.bw;
  }
  g.nbh = (g.H + g.bh - 1) / g.bh;
  g.nbw = (g.W + g.bw - 1) / g.bw;
  g.nbt = (g.T + g.bt - 1) / g.bt;
  g.HH = g.bh + g.kh - 1;
  g.HW = g.bw + g.kw - 1;
  g.HT = g.bt + g.kt - 1;
  g.k = p.k;
  g.kp = p.kp;
  g.ktp = p.kp;
  if (wrap) {
    g.Hsrc = g.H;
    g.hoff = 0;
    g.wrapH = 1;
  } else {
    g.Hsrc = g.H + g.kh - 1;
    g.hoff = g.kh - 1;
    g.wrapH = 0;
  }
  return g;
}

inline size_t fwd_smem(const Geo& g) {
  return (2 * BK * BN + g.ktp + static_cast<size_t>(g.HH) * g.HW * g.HT) * 4;
}
inline size_t adj_smem(const Geo& g) {
  return (BK * (BM + 4) + 2 * BK * BN + g.kp + g.ktp +
          static_cast<size_t>(g.HH) * g.HW * g.HT) * 4;
}

void check_smem(size_t need) {
  if (need > 220 * 1024)
    invalid("icnnm_b200: halo brick too large for shared memory (" + std::to_string(need) +
            " bytes); kernel box too large");
}

template <class K>
void set_max_dyn_smem(K kernel, int optin) {
  cudaFuncAttributes a;
  CK(cudaFuncGetAttributes(&a, kernel));
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          optin - static_cast<int>(a.sharedSizeBytes)));
}

void set_smem_attrs() {
  static thread_local int done_dev = -1;
  int dev;
  CK(cudaGetDevice(&dev));
  if (done_dev == dev) return;
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  set_max_dyn_smem(icnnm_dev::icnnm_fwd_ffma, optin);
  set_max_dyn_smem(icnnm_dev::icnnm_adj_ffma, optin);
  set_max_dyn_smem(icnnm_dev::icnnm_gram_lags, optin);
  for (int v = 0; v < 3; ++v) {  // tf32x3, f16x3, f16x3 CTA pairs
    CK(cudaFuncSetAttribute(icnnm_dev::tc::fwd_kernel_ptr(v > 0, v > 1),
                            cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    CK(cudaFuncSetAttribute(icnnm_dev::tc::adj_kernel_ptr(v > 0, v > 1),
                            cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  }
  done_dev = dev;
}

// Brick-ordered row of voxel (h, w, t) in a launch geometry.
inline int64_t brick_row(const Geo& g, int64_t h, int64_t w, int64_t t) {
  int64_t b = (h / g.bh * g.nbw + w / g.bw) * g.nbt + t / g.bt;
  int64_t v = g.vmap ? ((w % g.bw) * g.bh + (h % g.bh)) * g.bt + (t % g.bt)
                     : ((h % g.bh) * g.bw + (w % g.bw)) * g.bt + (t % g.bt);
  return b * BM + v;
}

// K (k x k column-major, f64) -> Krm [ktp][kp] (K[s][j]) and KT [kp][ktp].
void pack_basis(const Problem& p, const double* Kcm, std::vector<float>& Krm,
                std::vector<float>& KT) {
  const int k = p.k, kp = p.kp;
  Krm.assign(static_cast<size_t>(kp) * kp, 0.f);
  KT.assign(static_cast<size_t>(kp) * kp, 0.f);
  for (int j = 0; j < k; ++j)
    for (int s = 0; s < k; ++s) {
      float v = static_cast<float>(Kcm[static_cast<size_t>(j) * k + s]);
      Krm[static_cast<size_t>(s) * kp + j] = v;
      KT[static_cast<size_t>(j) * kp + s] = v;
    }
}

// ---------------------------------------------------------------------------
// tcgen05 engine plan and B packing
// ---------------------------------------------------------------------------
struct TcPlan {
  int kp = 0, ntn = 0, nkc = 0, nlast = 0, wbase = 0, sa = 0;
  bool f16 = false;        // F16x3 engine (kind::f16) instead of TF32x3
  float bunscale = 1.f;    // F16x3: inverse of B's power-of-2 scale
  int vmap = 0;            // voxel order of the brick geometry (Geo::vmap; adjoint N order)
  int width(int nt) const { return std::min(wbase, kp - nt * wbase); }
};

inline bool is_tc(int engine) {
  return engine == ICNNM_ENGINE_TF32X3 || engine == ICNNM_ENGINE_F16X3;
}

// N-tiling of kp columns into ntn tiles of width <= NTMAX (multiples of 16),
// minimising the measured MMA cost: an M=128 kind::tf32 MMA takes
// max(64, N/2) cycles on B200 (tools/ubench/mma_rate.cu), so few wide tiles
// beat many narrow ones (k=405: 2x208 instead of 128+128+128+32 = -19% MMA
// time, half the MMA instructions).  TMEM: 2 accumulators of wbase columns +
// sa A stages of 2*KC columns <= 512.
TcPlan tc_plan(const Problem& p, bool f16 = false) {
  TcPlan best;
  best.f16 = f16;
  const int kp = p.kp_tc;
  double best_cost = 1e300;
  const int n0 = (kp + icnnm_dev::tc::NTMAX - 1) / icnnm_dev::tc::NTMAX;
  for (int ntn = n0; ntn <= n0 + 8; ++ntn) {
    const int wb = static_cast<int>(roundup((kp + ntn - 1) / ntn, 16));
    if (wb > icnnm_dev::tc::NTMAX) continue;
    const int nt_eff = (kp + wb - 1) / wb;
    double cost = 0;
    for (int i = 0; i < nt_eff; ++i) cost += std::max(64.0, std::min(wb, kp - i * wb) / 2.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best.kp = kp;
      best.ntn = nt_eff;
      best.wbase = wb;
      best.nlast = kp - (nt_eff - 1) * wb;
    }
  }
  best.nkc = kp / icnnm_dev::tc::KC;
  const int stage_cols = f16 ? icnnm_dev::tc::KC : 2 * icnnm_dev::tc::KC;
  // A stages: as many as TMEM leaves next to the two accumulators, up to a cap
  // (ICNNM_TC_SA in the experiments build)
  static const int sa_cap = env_knob("ICNNM_TC_SA", 6);
  best.sa = std::min(std::min(icnnm_dev::tc::SA, sa_cap), (512 - 2 * best.wbase) / stage_cols);
  return best;
}

// tcgen05 engine geometry.  ICNNM_TC_BT32=1 (experiment, off by default)
// uses 2 x 2 x 32 bricks when T is a multiple of 32, so that each warp's 32
// TMEM lanes are 32 consecutive t: halo gathers and the adjoint's col2im
// scatter become conflict-free (SMEM bank conflicts -65% / -83%), but the
// larger halo (3600 vs 2400 words per brick at config 2) and output-brick
// flush cost more than the conflicts did (forward +7%, adjoint +14%;
// profiles/README_r1.md).
Geo tc_geo(const Geo& g, const TcPlan& t) {
  Geo q = g;
  q.kp = t.kp;
  q.ktp = t.kp;
  static const bool bt32 = env_knob("ICNNM_TC_BT32", 0) == 1;
  if (bt32 && g.T % 32 == 0 && g.W >= 2 && g.H >= 2) {
    q.bt = 32;
    q.bw = 2;
    q.bh = BM / (q.bt * q.bw);
    q.nbh = (q.H + q.bh - 1) / q.bh;
    q.nbw = (q.W + q.bw - 1) / q.bw;
    q.nbt = (q.T + q.bt - 1) / q.bt;
    q.HH = q.bh + q.kh - 1;
    q.HW = q.bw + q.kw - 1;
    q.HT = q.bt + q.kt - 1;
  }
  // Voxel order within a brick.  A warp's 32 TMEM lanes are two runs of 16
  // consecutive t (bt = 16) one brick row apart: D = HT words (vmap 0, rows
  // differ in w) or HW*HT words (vmap 1, rows differ in h).  The halo gathers
  // and the adjoint's col2im scatter hit |16 - D mod 32| lanes in 2-way bank
  // conflicts; config 2 (HT = 20, HW*HT = 240): 4 vs 0.  vmap 1 needs bh*bt = 32
  // (a warp then shares vw; the adjoint's N order becomes sw-fastest).
  q.vmap = 0;
  static const int vmap_env = env_knob("ICNNM_TC_VMAP", -1);
  if (q.bt == 16 && q.bh * q.bt == 32 && q.kw >= 1) {
    auto conf = [](int d) { return std::abs(16 - (d % 32)); };
    const bool better = conf(q.HW * q.HT) < conf(q.HT);
    q.vmap = vmap_env >= 0 ? (vmap_env != 0 ? 1 : 0) : (better ? 1 : 0);
  }
  return q;
}

inline float tf32_rna(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Pre-packed B tiles in the UMMA canonical SWIZZLE_NONE K-major layout, hi and
// lo TF32 parts: [nt][kc] blocks of 32 KB = [hl][q][n/8][k/4][n%8][k%4].
// forward: B(n=j, k=s) = K[s][j];  adjoint: B(n=s, k=j) = K[s][j].
// Adjoint N order (icnnm_tc.cu tapoff): n = (sw*kt + st)*kh + sh -> tap s.
// vmap 1 (warps share vw): n = (sh*kt + st)*kw + sw, sw fastest.
inline int adj_tap(const Problem& p, int n, int vmap) {
  const int kh = static_cast<int>(p.kd[0]), kw = static_cast<int>(p.kd[1]),
            kt = static_cast<int>(p.kd[2]);
  if (vmap) {
    const int sw = n % kw, q = n / kw, st = q % kt, sh = q / kt;
    return (sh * kw + sw) * kt + st;
  }
  const int sh = n % kh, q = n / kh, st = q % kt, sw = q / kt;
  return (sh * kw + sw) * kt + st;
}

// F16x3 B tiles: per (nt, kc) block [hl][n/8][k/8][n%8][k%8] halves of
// s * B (s = 2^eB puts max|K| below 2^14), hi = rn_f16(s x), lo = rn_f16(s x - hi);
// the lo block starts wn * 16 halves after hi.  Same block stride as TF32x3.
std::vector<float> pack_b_tiles_f16(const Problem& p, TcPlan& t, const double* Kcm, bool fwd) {
  const int k = p.k;
  double amax = 0.0;
  for (size_t i = 0; i < static_cast<size_t>(k) * k; ++i) amax = std::max(amax, std::fabs(Kcm[i]));
  int ex = 0;
  if (amax > 0) std::frexp(amax, &ex);
  const int eb = 14 - ex;
  t.bunscale = static_cast<float>(std::ldexp(1.0, -eb));
  const int blk = icnnm_dev::tc::B_STAGE_BYTES / 4;
  std::vector<float> out(static_cast<size_t>(t.ntn) * t.nkc * blk, 0.f);
  for (int nt = 0; nt < t.ntn; ++nt) {
    const int wn = t.width(nt);
    for (int kc = 0; kc < t.nkc; ++kc) {
      __half* base = reinterpret_cast<__half*>(out.data() + (static_cast<size_t>(nt) * t.nkc + kc) * blk);
      for (int n = 0; n < wn; ++n)
        for (int k16 = 0; k16 < icnnm_dev::tc::KC; ++k16) {
          const int nn = nt * t.wbase + n;
          const int kk = kc * icnnm_dev::tc::KC + k16;
          double x = 0.0;
          if (nn < k && kk < k)
            x = fwd ? Kcm[static_cast<size_t>(nn) * k + kk]
                    : Kcm[static_cast<size_t>(kk) * k + adj_tap(p, nn, t.vmap)];
          const float xs = static_cast<float>(std::ldexp(x, eb));
          const __half hi = __float2half_rn(xs);
          const __half lo = __float2half_rn(xs - __half2float(hi));
          const size_t off = (n / 8) * 128 + (k16 / 8) * 64 + (n % 8) * 8 + (k16 % 8);
          base[off] = hi;
          base[static_cast<size_t>(wn) * 16 + off] = lo;
        }
    }
  }
  return out;
}

// The same F16x3 tiles packed on the device from an f64 copy of K (one thread
// per tile element; bit-identical to pack_b_tiles_f16: x * 2^eB is exact in
// f64, then one rounding to f32 and the two RN conversions to f16).
__global__ void icnnm_pack_b_f16(int k, int kp, int wbase, int nkc, int kh, int kw, int kt,
                                 int fwd, int vmap, double sc, const double* __restrict__ K,
                                 __half* __restrict__ out, int64_t total) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int k16 = static_cast<int>(i % icnnm_dev::tc::KC);
  int64_t q = i / icnnm_dev::tc::KC;
  const int n = static_cast<int>(q % wbase);
  q /= wbase;
  const int kc = static_cast<int>(q % nkc);
  const int nt = static_cast<int>(q / nkc);
  const int wn = min(wbase, kp - nt * wbase);
  if (n >= wn) return;
  const int nn = nt * wbase + n;
  const int kk = kc * icnnm_dev::tc::KC + k16;
  double x = 0.0;
  if (nn < k && kk < k) {
    if (fwd) {
      x = K[static_cast<size_t>(nn) * k + kk];
    } else {
      int sh, sw, st;
      if (vmap) {
        sw = nn % kw;
        const int r = nn / kw;
        st = r % kt;
        sh = r / kt;
      } else {
        sh = nn % kh;
        const int r = nn / kh;
        st = r % kt;
        sw = r / kt;
      }
      x = K[static_cast<size_t>(kk) * k + (sh * kw + sw) * kt + st];
    }
  }
  const float xs = static_cast<float>(x * sc);
  const __half hi = __float2half_rn(xs);
  const __half lo = __float2half_rn(xs - __half2float(hi));
  __half* base = out + (static_cast<size_t>(nt) * nkc + kc) * (icnnm_dev::tc::B_STAGE_BYTES / 2);
  const size_t off = (n / 8) * 128 + (k16 / 8) * 64 + (n % 8) * 8 + (k16 % 8);
  base[off] = hi;
  base[static_cast<size_t>(wn) * 16 + off] = lo;
}

void pack_b_tiles_f16_device(const Problem& p, TcPlan& t, const double* dK, bool fwd,
                             DBuf<float>& out, cudaStream_t stream) {
  const int blk = icnnm_dev::tc::B_STAGE_BYTES / 4;
  out.alloc(static_cast<size_t>(t.ntn) * t.nkc * blk);
  CK(cudaMemsetAsync(out.p, 0, out.bytes(), stream));
  const int eb = static_cast<int>(std::lround(-std::log2(static_cast<double>(t.bunscale))));
  const int64_t total = static_cast<int64_t>(t.ntn) * t.nkc * t.wbase * icnnm_dev::tc::KC;
  icnnm_pack_b_f16<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(
      p.k, t.kp, t.wbase, t.nkc, static_cast<int>(p.kd[0]), static_cast<int>(p.kd[1]),
      static_cast<int>(p.kd[2]), fwd ? 1 : 0, t.vmap, std::ldexp(1.0, eb), dK,
      reinterpret_cast<__half*>(out.p), total);
  CKL();
}

// B's power-of-2 scale for F16x3 (max|K| below 2^14): sets t.bunscale = 2^-eB.
void f16_basis_scale(const Problem& p, TcPlan& t, const double* Kcm) {
  double amax = 0.0;
  for (size_t i = 0; i < static_cast<size_t>(p.k) * p.k; ++i) amax = std::max(amax, std::fabs(Kcm[i]));
  int ex = 0;
  if (amax > 0) std::frexp(amax, &ex);
  t.bunscale = static_cast<float>(std::ldexp(1.0, -(14 - ex)));
}

std::vector<float> pack_b_tiles(const Problem& p, TcPlan& t, const double* Kcm, bool fwd) {
  if (t.f16) return pack_b_tiles_f16(p, t, Kcm, fwd);
  const int k = p.k;
  const int blk = icnnm_dev::tc::B_STAGE_BYTES / 4;
  std::vector<float> out(static_cast<size_t>(t.ntn) * t.nkc * blk, 0.f);
  for (int nt = 0; nt < t.ntn; ++nt) {
    const int wn = t.width(nt);
    for (int kc = 0; kc < t.nkc; ++kc) {
      float* base = out.data() + (static_cast<size_t>(nt) * t.nkc + kc) * blk;
      for (int q = 0; q < icnnm_dev::tc::KC / 8; ++q)
        for (int n = 0; n < wn; ++n)
          for (int k8 = 0; k8 < 8; ++k8) {
            const int nn = nt * t.wbase + n;
            const int kk = kc * icnnm_dev::tc::KC + q * 8 + k8;
            double x = 0.0;
            if (nn < k && kk < k)
              x = fwd ? Kcm[static_cast<size_t>(nn) * k + kk]
                      : Kcm[static_cast<size_t>(kk) * k + adj_tap(p, nn, t.vmap)];
            const float xf = static_cast<float>(x);
            const float hi = tf32_rna(xf);
            const float lo = xf - hi;
            const size_t off = static_cast<size_t>(q) * (8 * wn) + (n / 8) * 64 + (k8 / 4) * 32 +
                               (n % 8) * 4 + (k8 % 4);
            base[off] = hi;
            base[(icnnm_dev::tc::KC / 8) * 8 * wn + off] = lo;
          }
    }
  }
  return out;
}

inline int64_t tc_w_elems(const Geo& g, const TcPlan& t) {
  return n_bricks(g) * static_cast<int64_t>(t.kp) * 128;
}

// 2-D tensor map (rows of 32 B = 16 halves) over a packed F16x3 B buffer with a
// box of `rows` rows, for the CTA pairs' .cta_group::2 tensor copies.  Encoded
// through the runtime's driver entry point (no libcuda link); cached per
// (buffer, box).
CUtensorMap pair_b_map(const float* Bpk, const TcPlan& t, int rows) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      fail(ICNNM_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<Encode>(fn);
  }();
  static std::map<std::tuple<const float*, int, int>, CUtensorMap> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  const int64_t total_rows =
      static_cast<int64_t>(t.ntn) * t.nkc * (icnnm_dev::tc::B_STAGE_BYTES / 32);
  auto key = std::make_tuple(Bpk, rows, static_cast<int>(total_rows));
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap m{};
  const cuuint64_t dims[2] = {16, static_cast<cuuint64_t>(total_rows)};
  const cuuint64_t strides[1] = {32};
  const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<float*>(Bpk), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ICNNM_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  cache.emplace(key, m);
  return m;
}

// Launch configuration of one tcgen05 kernel: knobs, tile groups, CTA pairs /
// multicast, split + resident-B mode, shared-memory carve-up and grid.  Pure
// function of the geometry and plan (the solver also uses it to size the
// deterministic adjoint's scratch before capturing its graphs).
struct TcConfig {
  icnnm_dev::tc::TcArgs a{};
  unsigned grid = 0;
  size_t smem = 0;
  bool cluster = false;  // 2-CTA clusters (pairs / B multicast)
  void* fn = nullptr;
};

TcConfig tc_config(const Geo& gtc, const TcPlan& t, bool fwd, bool have_b, bool no_auto_pairs = false) {
  TcConfig cfg;
  icnnm_dev::tc::TcArgs& a = cfg.a;
  a.bunscale = t.bunscale;
  static const int skip_env = env_knob("ICNNM_TC_SKIP", 0);  // timing experiments only (results invalid)
  a.skip = skip_env;
  static const int warr_env = env_knob("ICNNM_TC_WARR", 1);
  a.warr = warr_env;
  static const int bsplit_env = env_knob("ICNNM_TC_BSPLIT", 0);
  a.bsplit = bsplit_env;
  static const int bpair_env = env_knob("ICNNM_TC_BPAIR", 0);
  a.bpair = bpair_env;
  a.g = gtc;
  a.ntn = t.ntn;
  a.nkc = t.nkc;
  a.nlast = t.nlast;
  a.wbase = t.wbase;
  a.accw = t.wbase;
  a.sa = t.sa;
  // Tile groups (icnnm_tc.cu tg_seq): pairs of N-tiles share every built A
  // chunk (half the A-operand builds and, in the adjoint, half the W-chunk
  // loads).  The skew needs spare A stages beyond D, so it is used only when
  // the plan leaves at least 4 (F16x3 at k = 405: 6 stages).  Measured on the
  // same box (config 2, profiles/ab_r1/README.md): the adjoint gains (0.76 ->
  // 0.73 ms), the forward loses (0.70 -> 0.77 ms: its heavier epilogue is no
  // longer hidden behind the other tile's MMAs), so only the adjoint pairs.
  // ICNNM_TC_GRP / ICNNM_TC_SKEW override both kernels for A/B experiments.
  static const int grp_env = env_knob("ICNNM_TC_GRP", -1);
  static const int skew_env = env_knob("ICNNM_TC_SKEW", -1);
  const bool can_pair = t.ntn >= 2 && t.sa >= 4;
  a.grp = grp_env >= 0 ? grp_env : ((can_pair && !fwd) ? 2 : 1);
  a.skew = skew_env >= 0 ? skew_env : std::max(0, t.sa - 2);
  // deepest (B, W) stage counts that fit in shared memory (227 KB opt-in).
  // W depth is even: the two builder groups own alternate K-chunks, so with an
  // even ring each W stage is only ever consumed by one group.  With an odd
  // ring consecutive uses of a stage alternate between groups, and a group
  // running two uses ahead (possible with F16x3's 6 A stages) would pass its
  // parity wait on the previous fill.
  // CTA pairs (F16x3): thread-block clusters of 2 on one TPC run cta_group::2
  // MMAs (M = 256, one per pair): each CTA builds its own brick's A in its own
  // TMEM but loads only half of every B tile (N split across the pair), so the
  // B stream -- 13.3 KB per 312-cycle chunk and SM, the largest L2 and SMEM
  // consumer (and a quarter of the board power, profiles/ab_r1) -- halves.
  // With a streamed B they are on par with single CTAs (DESIGN 11), so the
  // default uses them only where they change what fits in shared memory: the
  // adjoint of a basis that single CTAs can keep resident only as two N-tile
  // roles (each building the brick's A operand, flushing its own output box and
  // streaming W again) but a pair keeps resident as halves with whole bricks per
  // CTA (config 4: adjoint 0.295 -> 0.249 ms; the forward, whose tiles do not
  // share built chunks, loses 11% and stays on single CTAs).
  // ICNNM_TC_CS=1|2 (experiments build) forces single CTAs / pairs for both kernels.
  static const int cs_env = env_knob("ICNNM_TC_CS", -1);
#ifndef ICNNM_DEFAULT_CS
#define ICNNM_DEFAULT_CS 1  // build-time A/B: 2 = CTA pairs wherever they are possible
#endif
  a.cs = cs_env >= 0 ? cs_env : ICNNM_DEFAULT_CS;
  bool auto_pairs = false;
#ifndef ICNNM_FWD_PAIRS
#define ICNNM_FWD_PAIRS 0  // build-time A/B: the forward on resident pairs too
#endif
  if (cs_env < 0 && !no_auto_pairs && (!fwd || ICNNM_FWD_PAIRS) && t.f16 && have_b &&
      env_knob("ICNNM_TC_BRES", -1) != 0) {
    const int full = t.ntn * t.nkc * t.wbase * icnnm_dev::tc::KC * 4;
    const bool single_fits =
        icnnm_dev::tc::smem_bytes(gtc, fwd, 1, 4, true, false, 1, full, 2) <= 227 * 1024;
    const bool pair_fits =
        icnnm_dev::tc::smem_bytes(gtc, fwd, 1, 4, true, true, 1, full / 2, 2) <= 227 * 1024;
    if (!single_fits && pair_fits && t.ntn >= 2 && t.sa >= 4) {
      a.cs = 2;
      auto_pairs = true;
    }
  }
  if (!t.f16 || n_bricks(gtc) < 2) a.cs = 1;
  const bool pairs = a.cs > 1;
  // pairs: the peer's half of every B stage signals the leader's barrier
  // directly through 2-SM tensor copies (ICNNM_TC_TMAPAIR=0: bulk copies and a
  // relay thread, the first pair design)
  static const int tmapair_env = env_knob("ICNNM_TC_TMAPAIR", 1);
  a.tma_pair = (pairs && tmapair_env != 0 && have_b) ? 1 : 0;
  // B multicast (F16x3 single CTAs in 2-CTA clusters sharing one B stream, each
  // CTA loading half of every stage): ICNNM_TC_MCB=1 (A/B experiment)
  static const int mcb_env = env_knob("ICNNM_TC_MCB", 0);
  a.mcb = (mcb_env > 0 && t.f16 && !pairs && n_bricks(gtc) >= 2) ? 1 : 0;
  // F16x3 B stages are 16 KB (half the TF32 stage), which leaves room for
  // an 8-deep forward W-group ring: a 208-column tile has 8 W groups, so the
  // whole tile's W_old is in flight before its epilogue starts.  Deepest B
  // ring up to the cap first, then the deepest even W ring that still fits.
  // 4 B stages measured faster than 5-6 for TF32x3 (more SMEM leaves less L1):
  // profiles/README_r1.md; CTA pairs hold half-size stages, so twice as many
  // in the same space
  static const int sb_env = env_knob("ICNNM_TC_SB", -1);
  // F16x3 single CTAs: 8 stages (+1.8% / +1.3% over 4 / 6 on config 2,
  // profiles/ab_r1/tune/, profiles/ab_r1/sb8/)
  // (round 2: the F16x3 forward keeps 6 -- the shared memory of two more B
  // stages holds two more 16 KB W-group stages, and the epilogue's W_old loads,
  // not the B ring, are what its MMA warp ends up waiting for: config 2 forward
  // 0.606 -> 0.583 ms, config 3 28.2 -> 28.1 ms; the adjoint loses with fewer)
  const int sb_cap = sb_env > 0 ? sb_env : (pairs ? 8 : (t.f16 ? (fwd ? 6 : 8) : 4));
  static const int ws_cap = env_knob("ICNNM_TC_WS", icnnm_dev::tc::WS);
  // Adjoint epilogue: a second 4-warp half (alternate 32-column blocks, its
  // own 4 output bricks) when those bricks fit next to a B ring of >= 4
  // stages; otherwise one half.  ICNNM_TC_EHALF=1|2 overrides (A/B).
  static const int eh_env = env_knob("ICNNM_TC_EHALF", -1);
  a.sb = 2;
  a.ws = 2;
  a.ehalf = 1;
  a.nsplit = 1;
  a.bres = 0;
  a.bres_stride = 0;
  a.bres_bytes = 0;
  a.bmix = 0;
  a.nresblk = 0;
  bool found = false;
  // Resident B (F16x3 single CTAs): when the basis tiles of one CTA role fit
  // in shared memory next to a W ring of >= 4 stages, they are loaded once
  // per launch instead of once per brick -- the per-brick B stream (the whole
  // hi/lo basis, e.g. 256 KB at k = 245) disappears from L2 and SMEM.  A
  // brick's work is split over nsplit CTA roles by N-tiles when the whole
  // basis does not fit (forward: each role its own columns of W; adjoint: its
  // own taps, partial output bricks summed by the flush).
  // Measured at config 4 (k = 245, 2 N-tiles; profiles/r2/README.md): the
  // adjoint gains 8% (0.406 -> 0.375 ms: its MMA waited on B 45% of the
  // time) and, with the halo-preparation warps taking the per-brick halo
  // work off the builders, the forward 10% (0.347 -> 0.312 ms).
  // ICNNM_TC_BRES=0|1 (experiments build) forces it off / on.
  static const int bres_env = env_knob("ICNNM_TC_BRES", -1);
  const bool bres_on = bres_env != 0;
  // forward: halo buffers for the prep warps' software pipeline (4: they run
  // two bricks ahead of the builders), fewer when shared memory is short
  static const int nhb_env = env_knob("ICNNM_TC_NHB", icnnm_dev::tc::NHB_MAX);
  for (int nhb = fwd ? std::min(nhb_env, icnnm_dev::tc::NHB_MAX) : 2; nhb >= 2 && !found; --nhb) {
  a.nhb = nhb;
  // Mixed residency (adjoint with tile groups): whole bricks per CTA -- the A
  // operand (W c -> f16 hi/lo, the largest instruction item of the adjoint) is
  // built once per brick and the col2im output box flushed once, instead of
  // once per N-tile role -- with as many (tile, chunk) blocks of B resident
  // as fit next to a tight ring of >= 3 stages for the rest.  Chosen when the
  // whole basis does not fit (it does at ns = 1 only for small k) but at
  // least a quarter of it does.  Measured at config 4: the halved builder and
  // flush work is paid back by the MMA warp waiting on the half-streamed B
  // (35% of its time; adjoint 0.362 vs 0.342 ms), so the mode is opt-in:
  // ICNNM_TC_BMIX=1 (experiments build).
  static const int bmix_env = env_knob("ICNNM_TC_BMIX", 0);  // measured slower (profiles/r2/README.md): opt-in
  static const int bmix_sb = env_knob("ICNNM_TC_BMIX_SB", 4);
  static const int bmix_ws = env_knob("ICNNM_TC_BMIX_WS", 4);
  static const int bmix_eh = env_knob("ICNNM_TC_BMIX_EH", 2);
  if (t.f16 && !pairs && !a.mcb && have_b && bres_on && !fwd && a.grp == 2 && bmix_env > 0) {
    const int stride = t.wbase * icnnm_dev::tc::KC * 4;
    const int nblk = t.ntn * t.nkc;
    const int sbv = std::max(3, std::min(bmix_sb, icnnm_dev::tc::SB - 1));
    const int wsv = std::max(4, std::min(bmix_ws, icnnm_dev::tc::WS) & ~1);
    for (int eh = std::min(2, std::max(1, bmix_eh)); eh >= 1 && !found; --eh) {
      const size_t base = icnnm_dev::tc::smem_bytes(gtc, fwd, sbv, wsv, t.f16, false, eh, 0, nhb, stride);
      if (base >= 227 * 1024) continue;
      const int fit = static_cast<int>((227 * 1024 - base) / stride);
      // every block resident is the plain resident mode's business (below)
      if (fit >= nblk || fit * 4 < nblk) continue;
      a.nsplit = 1;
      a.bres = 1;
      a.bmix = 1;
      a.nresblk = fit & ~1;  // chunk pairs are resident or streamed together
      a.bres_stride = stride;
      a.bres_bytes = a.nresblk * stride;
      a.sb = sbv;
      a.ws = wsv;
      a.ehalf = eh;
      a.bstride = stride;
      found = true;
    }
  }
  // CTA pairs with resident B: each CTA keeps its half of every tile's N rows
  // (hi half, lo half), so a basis that needs two N-tile roles as single CTAs
  // (config 4: 256 KB) is resident with whole bricks per CTA -- A built once
  // per brick, one output-box flush, one W stream -- and no B ring at all.
  if (!found && t.f16 && pairs && have_b && bres_on) {
    const int stride = t.wbase * icnnm_dev::tc::KC * 4 / 2;
    const int need = t.ntn * t.nkc * stride;
    for (int eh = fwd ? 1 : 2; eh >= 1 && !found; --eh)
      for (int wsv = std::min(ws_cap, icnnm_dev::tc::WS) & ~1; wsv >= 4 && !found; wsv -= 2)
        if (icnnm_dev::tc::smem_bytes(gtc, fwd, 1, wsv, t.f16, true, eh, need, nhb) <= 227 * 1024) {
          a.nsplit = 1;
          a.bres = 1;
          a.bres_stride = stride;
          a.bres_bytes = need;
          a.sb = 1;
          a.ws = wsv;
          a.ehalf = eh;
          found = true;
        }
  }
  if (!found && t.f16 && !pairs && !a.mcb && have_b && bres_on) {
    const int stride = t.wbase * icnnm_dev::tc::KC * 4;
    for (int ns = 1; ns <= 4 && !found; ++ns) {
      if (ns > t.ntn) break;
      int maxb = 0;
      for (int r = 0; r < ns; ++r) {
        const int ntiles = (r + 1) * t.ntn / ns - r * t.ntn / ns;
        maxb = std::max(maxb, ntiles * t.nkc * stride);
      }
      for (int eh = fwd ? 1 : 2; eh >= 1 && !found; --eh)
        for (int wsv = std::min(ws_cap, icnnm_dev::tc::WS) & ~1; wsv >= 4 && !found; wsv -= 2)
          if (icnnm_dev::tc::smem_bytes(gtc, fwd, 1, wsv, t.f16, false, eh, maxb, nhb) <=
              227 * 1024) {
            a.nsplit = ns;
            a.bres = 1;
            a.bres_stride = stride;
            a.bres_bytes = maxb;
            a.sb = 1;
            a.ws = wsv;
            a.ehalf = eh;
            found = true;
          }
    }
  }
  // tight B stages (ICNNM_TC_BTIGHT=1, experiments): the ring's stage stride is
  // the widest tile's bytes (8 KB at k = 245 instead of 16 KB), so the same
  // shared memory holds up to twice as many chunks of lookahead
  static const int btight_env = env_knob("ICNNM_TC_BTIGHT", 0);
  const bool tight = t.f16 && !pairs && btight_env != 0;
  if (!a.bmix) a.bstride = tight ? t.wbase * icnnm_dev::tc::KC * 4 : 0;
  const int sbc = tight ? std::max(sb_cap, icnnm_dev::tc::B_STAGE_F16 / std::max(1, a.bstride) * sb_cap)
                        : sb_cap;
  for (int eh = fwd ? 1 : (eh_env > 0 ? eh_env : 2); eh >= 1 && !found; --eh) {
    const int sb_min = (eh == 2 && eh_env <= 0) ? std::min(4, sbc) : 2;
    for (int sbv = std::min(sbc, icnnm_dev::tc::SB); sbv >= sb_min && !found; --sbv)
      for (int wsv = std::min(ws_cap, icnnm_dev::tc::WS) & ~1; wsv >= 2 && !found; wsv -= 2)
        if (icnnm_dev::tc::smem_bytes(gtc, fwd, sbv, wsv, t.f16, pairs, eh, 0, nhb, a.bstride) <=
            227 * 1024) {
          a.sb = sbv;
          a.ws = wsv;
          a.ehalf = eh;
          found = true;
        }
  }
  }  // nhb
  icnnm_dev::tc::tc_fill_taps(a, fwd);
  a.nbricks = n_bricks(gtc);
  int dev = 0, nsm = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  cfg.smem = icnnm_dev::tc::smem_bytes(gtc, fwd, a.sb, a.ws, t.f16, pairs, a.ehalf, a.bres_bytes,
                                       a.nhb, (a.bres && !a.bmix) ? 0 : a.bstride, a.bmix != 0);
  if (cfg.smem > 227 * 1024) invalid("icnnm_b200: tcgen05 engine shared memory exceeds 227 KB");
  cfg.fn = fwd ? icnnm_dev::tc::fwd_kernel_ptr(t.f16, a.cs > 1)
               : icnnm_dev::tc::adj_kernel_ptr(t.f16, a.cs > 1);
  cfg.cluster = a.cs > 1 || a.mcb;
  if (cfg.cluster) {
    // persistent grid: as many 2-CTA clusters as can be co-resident (one GPC each)
    static std::map<std::pair<void*, size_t>, int> max_pairs;
    static std::mutex mp_mu;
    std::lock_guard<std::mutex> lk(mp_mu);
    auto key = std::make_pair(cfg.fn, cfg.smem);
    auto it = max_pairs.find(key);
    if (it == max_pairs.end()) {
      cudaLaunchConfig_t qc{};
      cudaLaunchAttribute at{};
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = 2;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      qc.gridDim = dim3(static_cast<unsigned>(nsm));
      qc.blockDim = dim3(icnnm_dev::tc::threads(fwd));
      qc.dynamicSmemBytes = cfg.smem;
      qc.attrs = &at;
      qc.numAttrs = 1;
      int n = 0;
      CK(cudaOccupancyMaxActiveClusters(&n, cfg.fn, &qc));
      it = max_pairs.emplace(key, std::max(1, n)).first;
    }
    const int64_t nslot = (a.nbricks + 1) / 2;
    // a device on which fewer than 80% of the SMs can run as co-resident pairs
    // (disabled SMs splitting TPCs) keeps the automatic choice on single CTAs
    if (auto_pairs && a.cs > 1 && 2 * it->second * 5 < nsm * 4 && nslot > it->second)
      return tc_config(gtc, t, fwd, have_b, true);
    cfg.grid = 2u * static_cast<unsigned>(std::min<int64_t>(nslot, it->second));
  } else {
    // split mode: a multiple of nsplit CTAs, role = blockIdx % nsplit
    const int64_t want = std::min<int64_t>(a.nbricks * a.nsplit, nsm);
    cfg.grid = static_cast<unsigned>(std::max<int64_t>(a.nsplit, want / a.nsplit * a.nsplit));
  }
  return cfg;
}

void launch_tc_kernel(const Geo& gtc, const TcPlan& t, bool fwd, int mode, const float* src,
                      float* W, const float* Bpk, const float* cvec, float* adj, double* norm2,
                      const IterState* st, cudaStream_t stream,
                      unsigned long long* dbg = nullptr, float amax = 0.f, bool pdl = false,
                      float2* adjq = nullptr, double* npart = nullptr) {
  TcConfig cfg = tc_config(gtc, t, fwd, Bpk != nullptr);
  icnnm_dev::tc::TcArgs& a = cfg.a;
  a.amax = amax;
  a.dbg = dbg;
  a.src = src;
  a.Win = W;
  a.Wout = W;
  a.Bpk = Bpk;
  a.cvec = cvec;
  a.adj = adj;
  a.norm2 = norm2;
  a.st = st;
  a.mode = mode;
  a.adjq = adjq;
  a.npart = npart;
  if (a.tma_pair) {
    a.tmB[0] = pair_b_map(Bpk, t, t.wbase / 2);
    a.tmB[1] = pair_b_map(Bpk, t, std::max(8, t.nlast / 2));
  }
  void* args[] = {&a};
  const dim3 block(icnnm_dev::tc::threads(fwd));
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute at[2]{};
  lc.gridDim = dim3(cfg.grid);
  lc.blockDim = block;
  lc.dynamicSmemBytes = cfg.smem;
  lc.stream = stream;
  lc.attrs = at;
  lc.numAttrs = 0;
  if (cfg.cluster) {
    at[lc.numAttrs].id = cudaLaunchAttributeClusterDimension;
    at[lc.numAttrs].val.clusterDim.x = 2;
    at[lc.numAttrs].val.clusterDim.y = 1;
    at[lc.numAttrs].val.clusterDim.z = 1;
    ++lc.numAttrs;
  }
  if (pdl) {
    at[lc.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[lc.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++lc.numAttrs;
  }
  CK(cudaLaunchKernelExC(&lc, cfg.fn, args));
}

// EigenBasis::validate (spectral.cpp:25-41), run on every call that takes a
// basis, as the reference runs it inside every icnnm_solve (solver.cpp:154);
// the handle API validates once at create (BasisConvolver's precompute-once
// pattern, conv_op.hpp:61-64).
void validate_orthogonal(int k, const double* K);
void validate_evals(int k, const double* evals);

void validate_basis(int k, const double* K, const double* evals) {
  if (!K) invalid("EigenBasis: K must be k x k");
  validate_orthogonal(k, K);
  validate_evals(k, evals);
}

void validate_orthogonal(int k, const double* K) {
  // max |K^T K - I| over the lower triangle, four independent partial sums per
  // dot product (the check is a 1e-10 tolerance, so summation order is free);
  // rows interleaved over up to 8 host threads for large k
  auto rows = [&](int t0, int step) {
    double worst = 0.0;
    for (int i = t0; i < k; i += step) {
      const double* ci = K + static_cast<size_t>(i) * k;
      for (int j = 0; j <= i; ++j) {
        const double* cj = K + static_cast<size_t>(j) * k;
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
        int r = 0;
        for (; r + 4 <= k; r += 4) {
          d0 += ci[r] * cj[r];
          d1 += ci[r + 1] * cj[r + 1];
          d2 += ci[r + 2] * cj[r + 2];
          d3 += ci[r + 3] * cj[r + 3];
        }
        for (; r < k; ++r) d0 += ci[r] * cj[r];
        double d = (d0 + d1) + (d2 + d3);
        if (i == j) d -= 1.0;
        if (!(std::fabs(d) <= worst)) worst = std::isnan(d) ? HUGE_VAL : std::fabs(d);
      }
    }
    return worst;
  };
  const int nth = k >= 128 ? static_cast<int>(std::max(1u, std::min(8u, std::thread::hardware_concurrency()))) : 1;
  std::vector<double> part(nth, 0.0);
  std::vector<std::thread> pool;
  for (int t = 1; t < nth; ++t) pool.emplace_back([&, t] { part[t] = rows(t, nth); });
  part[0] = rows(0, nth);
  for (auto& th : pool) th.join();
  double worst = 0.0;
  for (double w : part) worst = std::max(worst, w);
  if (!(worst <= 1e-10)) invalid("EigenBasis: K is not orthogonal");
}

void validate_evals(int k, const double* evals) {
  if (evals) {
    for (int i = 0; i < k; ++i) {
      if (evals[i] < 0) invalid("EigenBasis: negative eigenvalue");
      if (i > 0 && evals[i] > evals[i - 1] + 1e-12)
        invalid("EigenBasis: eigenvalues not nonincreasing");
    }
  }
}

void validate_cfg(const icnnm_solver_config* c) {
  if (!c) invalid("SolverConfig: null");
  if (!(c->lambda > 0)) invalid("SolverConfig: lambda must be > 0");
  if (c->has_theta0 && !(c->theta0 > 0)) invalid("SolverConfig: theta0 must be > 0");
  if (!(c->theta_growth >= 1)) invalid("SolverConfig: theta_growth must be >= 1");
  if (!(c->theta_max > 0)) invalid("SolverConfig: theta_max must be > 0");
  if (c->has_theta0 && c->theta0 > c->theta_max)
    invalid("SolverConfig: theta0 must be <= theta_max");
  if (c->max_iters < 1) invalid("SolverConfig: max_iters must be >= 1");
  if (!(c->tol_primal > 0) || !(c->tol_change > 0) || !(c->rank_tol > 0))
    invalid("SolverConfig: tolerances must be > 0");
  if (c->init_fill != ICNNM_INIT_ZERO && c->init_fill != ICNNM_INIT_MEAN)
    invalid("SolverConfig: init_fill must be 'zero' or 'mean'");
  if (c->engine != ICNNM_ENGINE_FFMA && !is_tc(c->engine) && c->engine != ICNNM_ENGINE_F64 &&
      c->engine != ICNNM_ENGINE_AUTO)
    invalid("SolverConfig: unknown engine");
}

// ICNNM_ENGINE_AUTO (include/icnnm_b200.h): the fp32 engines cannot resolve
// l_change below ~1e-7 (Delta carries the GEMMs' rounding) nor the primal
// residual below ~1e-4 (exact_residual) / ~3e-3 (identity), so a finite
// tolerance under those floors runs the fp64 engine; tolerances <= 1e-200
// count as disabled (fixed iteration counts).
icnnm_solver_config resolve_engine(const icnnm_solver_config& in) {
  icnnm_solver_config c = in;
  if (c.engine != ICNNM_ENGINE_AUTO) return c;
  const bool p_on = c.tol_primal > 1e-200, c_on = c.tol_change > 1e-200;
  if ((p_on && c.tol_primal < 1e-4) || (c_on && c.tol_change < 1e-6)) {
    c.engine = ICNNM_ENGINE_F64;
  } else {
    c.engine = ICNNM_ENGINE_F16X3;
    if (p_on) c.exact_residual = 1;
  }
  return c;
}


// ---------------------------------------------------------------------------
// Solver: one or more H-slabs of one tensor on this process' device.
// ---------------------------------------------------------------------------
struct Slab {
  int64_t row0 = 0, rows = 0;   // own rows [row0, row0 + rows)
  Geo g{};
  Geo gtc{};                    // tcgen05 engine geometry (kp = ktp = kp_tc)
  int64_t m_own = 0;            // rows * W * T
  int64_t halo_elems = 0;       // (kh-1) * W * T (slab mode)
  DBuf<float> Lt, adj, pm, mask, W;
  DBuf<float> Lr;                 // exact-residual mode: L_{t+1} (fp32, with halo rows)
  DBuf<float2> adjq;              // deterministic adjoint: {hi, lo} fixed-grid pairs (adj's layout)
  DBuf<double> L, V;
};

struct Solver {
  Problem p;
  int device = 0;
  bool sharded = false;          // slab mode with explicit halos
  int G = 1, world = 1, rank = 0, local = 1;
  std::vector<Slab> slabs;
  std::unique_ptr<Comm> comm;    // cross-process exchange (world > 1)
  DBuf<float> Krm, KT, cvec;
  TcPlan tp, tp16;               // tcgen05 engines: TF32x3 / F16x3 plans
  DBuf<float> BpkF, BpkA;        // TF32x3: packed B tiles (fwd / adj)
  DBuf<float> BpkF16, BpkA16;    // F16x3: packed B tiles (fwd / adj)
  int engine = ICNNM_ENGINE_FFMA;  // engine of the current run
  bool exact_res = false;          // exact primal residual (one extra forward / iteration)
  DBuf<double> red;              // norm2 (kp) | update slot (8)
  DBuf<double> theta;
  DBuf<IterState> st;
  DBuf<IterStats> stats;
  DBuf<double> Mstage, maskstage;  // f64 staging of the current problem
  // Deterministic reductions (tcgen05 engines): per-CTA / per-block partial
  // rows, folded in a fixed order; slab i owns rows
  // [i * rows_per_slab, (i + 1) * rows_per_slab), unused rows stay zero.
  bool det = false;
  DBuf<double> npart, upart, gpart;
  int nsm = 148, upd_rows = 0;
  DBuf<float> xfer_send, xfer_recv;  // cross-process halo buffers
  DBuf<double> comb;                 // cross-rank combine of the upload scalars
  double h_comb[5] = {0, 0, 0, 0, 0};
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs = nullptr;
  double* h_theta = nullptr;  // pinned staging of the theta schedule (thread's pool)
  IterState* h_st = nullptr;  // pinned: [0] initial state, [1] state readback (pool)
  // host copies of the basis (validation happens once at create)
  std::vector<double> K;
  // per-problem scalars (from upload)
  bool uploaded = false;
  double pm_absmax = 0, pm_norm2 = 0, pm_sum = 0;
  int64_t observed = 0;
  int64_t launches = 0;
  bool profile = false;
  bool tc_counters = false;
  // head graph launched while the rest of the solve is captured (ICNNM_GRAPH_SPLIT=0: one graph)
  bool graph_split = env_knob("ICNNM_GRAPH_SPLIT", 1) != 0;
  double prof_ms[4] = {0, 0, 0, 0};
  DBuf<unsigned long long> dbg;  // 2 x DBG_SLOTS tcgen05 pipeline counters

  ~Solver() {
    // the buffers go back to the device cache: nothing may still use them
    if (stream) cudaStreamSynchronize(stream);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (evs) cudaEventDestroy(evs);
    if (stream) cudaStreamDestroy(stream);
  }
};

void solver_alloc(Solver& S) {
  const Problem& p = S.p;
  CK(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&S.ev0));
  CK(cudaEventCreate(&S.ev1));
  CK(cudaEventCreate(&S.evs));
  set_smem_attrs();
  g_timer.mark("stream/events/attrs");
  S.tp = tc_plan(p);
  S.tp16 = tc_plan(p, true);
  const int64_t WT = p.dims[1] * p.dims[2];
  for (auto& s : S.slabs) {
    s.g = make_geo(p, s.rows, !S.sharded);
    check_smem(fwd_smem(s.g));
    check_smem(adj_smem(s.g));
    s.m_own = s.rows * WT;
    s.halo_elems = S.sharded ? (p.kd[0] - 1) * WT : 0;
    s.Lt.alloc(s.m_own + s.halo_elems);
    s.adj.alloc(s.m_own + s.halo_elems);
    s.pm.alloc(s.m_own);
    s.mask.alloc(s.m_own);
    s.L.alloc(s.m_own);
    s.V.alloc(s.m_own);
    s.gtc = tc_geo(s.g, S.tp);
    S.tp.vmap = S.tp16.vmap = s.gtc.vmap;  // same brick shape in every slab
    check_smem(icnnm_dev::tc::smem_bytes(s.gtc, true, 2, 2, false));
    check_smem(icnnm_dev::tc::smem_bytes(s.gtc, false, 2, 2, false));
    s.W.alloc(std::max<int64_t>(n_bricks(s.g) * BM * p.kp, tc_w_elems(s.gtc, S.tp)));
    CK(cudaMemsetAsync(s.adj.p, 0, s.adj.bytes(), S.stream));
  }
  g_timer.mark("device buffers");
  const int kpmax = std::max(p.kp, S.tp.kp);
  S.cvec.alloc(kpmax);
  S.red.alloc(kpmax + 8);
  S.st.alloc(1);
  // staging of this process' own rows only (all slabs: the whole tensor)
  int64_t mtot = 0;
  for (auto& s : S.slabs) mtot += s.m_own;
  S.Mstage.alloc(mtot);
  S.maskstage.alloc(mtot);
  if (S.comm) {
    S.comb.alloc(8);
    S.xfer_send.alloc((p.kd[0] - 1) * WT + 1);
    S.xfer_recv.alloc((p.kd[0] - 1) * WT + 1);
  }
  CK(cudaStreamSynchronize(S.stream));
}

// Upload: validation of solver.cpp:66-72 / tensor.hpp:115-121, host scalars.
void solver_upload(Solver& S, const double* M, const double* mask) {
  if (!M || !mask) invalid("solve: null input");
  // this process' own rows (every slab of an unsharded or single-process solve)
  int64_t m = 0;
  for (auto& s : S.slabs) m += s.m_own;
  // The staging buffers are overwritten below before the scan has finished:
  // the handle holds no problem until this upload has validated (a rejected
  // upload leaves "no problem uploaded", never the previous problem's scalars
  // next to the rejected data).
  S.uploaded = false;
  // The validation scan (sequential: pm's sums feed theta0 / res_scale in the
  // reference's order) runs on a helper thread while this thread pushes the
  // pageable H2D copies; an invalid input is reported after both finish.
  double amax = 0, n2 = 0, sum = 0;
  int64_t obs = 0;
  const char* err = nullptr;
  std::thread scan([&] {
    for (int64_t i = 0; i < m; ++i) {
      const double mk = mask[i];
      if (mk != 0.0 && mk != 1.0) {
        err = "SamplingMask: entries must be 0 or 1";
        return;
      }
      if (!std::isfinite(M[i])) {
        err = "solve: observations: non-finite tensor entries";
        return;
      }
      if (mk == 1.0) {
        const double v = M[i];
        amax = std::max(amax, std::fabs(v));
        n2 += v * v;
        sum += v;
        ++obs;
      }
    }
  });
  cudaError_t e1 = cudaMemcpyAsync(S.Mstage.p, M, m * sizeof(double), cudaMemcpyHostToDevice,
                                   S.stream);
  cudaError_t e2 = e1 == cudaSuccess ? cudaMemcpyAsync(S.maskstage.p, mask, m * sizeof(double),
                                                       cudaMemcpyHostToDevice, S.stream)
                                     : e1;
  cudaError_t e3 = e2 == cudaSuccess ? cudaStreamSynchronize(S.stream) : e2;
  scan.join();
  if (S.comm) {
    // slab-local inputs: theta0 (max |pm|, solver.cpp:88-91), res_scale
    // (||pm||, :97), the mean fill (:83-86) and the empty-set / validity
    // checks (:68-72) are global -- combined over the ranks (max / sum);
    // an invalid slab fails every rank (no rank is left waiting in a
    // collective)
    CK(e3);
    double* h = S.h_comb;
    h[0] = amax;
    h[1] = err ? 1.0 : 0.0;
    h[2] = n2;
    h[3] = sum;
    h[4] = static_cast<double>(obs);
    CK(cudaMemcpyAsync(S.comb.p, h, 5 * sizeof(double), cudaMemcpyHostToDevice, S.stream));
    S.comm->allreduce_max(S.comb.p, 2, S.stream);
    S.comm->allreduce_sum(S.comb.p + 2, 3, S.stream);
    CK(cudaMemcpyAsync(h, S.comb.p, 5 * sizeof(double), cudaMemcpyDeviceToHost, S.stream));
    CK(cudaStreamSynchronize(S.stream));
    if (err) invalid(err);
    if (h[1] != 0.0) invalid("solve: invalid input on another rank");
    amax = h[0];
    n2 = h[2];
    sum = h[3];
    obs = static_cast<int64_t>(h[4] + 0.5);
  }
  if (err) invalid(err);
  CK(e3);
  if (obs == 0) invalid("solve: empty sampling set");
  S.pm_absmax = amax;
  S.pm_norm2 = n2;
  S.pm_sum = sum;
  S.observed = obs;
  S.uploaded = true;
}

// L~ halo exchange: slab g's last kh-1 own rows -> slab g+1's halo rows.
void exchange_lt(Solver& S, DBuf<float> Slab::*buf = &Slab::Lt) {
  if (!S.sharded) return;
  const size_t he = S.slabs[0].halo_elems;
  if (he == 0) return;
  const int nl = static_cast<int>(S.slabs.size());
  if (!S.comm) {
    for (int i = 0; i < nl; ++i) {
      const Slab& src = S.slabs[i];
      Slab& dst = S.slabs[(i + 1) % nl];
      CK(cudaMemcpyAsync((dst.*buf).p, (src.*buf).p + src.m_own, he * sizeof(float),
                         cudaMemcpyDeviceToDevice, S.stream));
    }
    return;
  }
  // local neighbours first, then the process boundary through the comm.
  for (int i = 0; i + 1 < nl; ++i)
    CK(cudaMemcpyAsync((S.slabs[i + 1].*buf).p, (S.slabs[i].*buf).p + S.slabs[i].m_own,
                       he * sizeof(float), cudaMemcpyDeviceToDevice, S.stream));
  const Slab& last = S.slabs[nl - 1];
  S.comm->shift_forward((last.*buf).p + last.m_own, (S.slabs[0].*buf).p, he, S.stream);
}

// Adjoint reverse halo: slab g's halo partials -> added to slab g-1's last rows.
void exchange_adj(Solver& S) {
  if (!S.sharded) return;
  const int64_t he = S.slabs[0].halo_elems;
  if (he == 0) return;
  const int nl = static_cast<int>(S.slabs.size());
  auto add = [&](float* dst, float* src) {
    icnnm_dev::icnnm_add_rows<<<grid_for(he, 256), 256, 0, S.stream>>>(he, dst, src);
    CKL();
    ++S.launches;
  };
  if (!S.comm) {
    for (int i = 0; i < nl; ++i) {
      Slab& src = S.slabs[i];
      Slab& dst = S.slabs[(i + nl - 1) % nl];
      add(dst.adj.p + dst.m_own, src.adj.p);
    }
    return;
  }
  for (int i = nl - 1; i >= 1; --i) {
    Slab& src = S.slabs[i];
    Slab& dst = S.slabs[i - 1];
    add(dst.adj.p + dst.m_own, src.adj.p);
  }
  // slab 0's partials go to the previous process; ours come from the next.
  Slab& first = S.slabs[0];
  Slab& last = S.slabs[nl - 1];
  S.comm->shift_backward(first.adj.p, S.xfer_recv.p, he, S.stream);
  CK(cudaMemsetAsync(first.adj.p, 0, he * sizeof(float), S.stream));
  add(last.adj.p + last.m_own, S.xfer_recv.p);
}

int engine_kp(const Solver& S);
int slab_index(const Solver& S, const Slab& s) { return static_cast<int>(&s - S.slabs.data()); }

// Debugging only (experiments build): ICNNM_F16_OFF=1 runs the F16x3 engine's adjoint in TF32x3,
// =2 its forward (isolates a kernel when bisecting a failure).
inline int f16_debug_mask() {
  static const int m = env_knob("ICNNM_F16_OFF", 0);  // bisection only
  return m;
}

// icnnm_update grid: one resident wave (SMs x resident blocks of 256), capped
// by the work (UPD_U elements per thread).
int update_grid(int64_t m) {
  static const int wave = [] {
    int dev = 0, nsm = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, icnnm_dev::icnnm_update, 256, 0);
    return nsm * std::max(1, per);
  }();
  const int64_t need = (m + 256 * icnnm_dev::UPD_U - 1) / (256 * icnnm_dev::UPD_U);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, wave)));
}

// The basis in the layout of one engine, packed and uploaded on the first run
// that uses the engine (an end-to-end call packs only what it runs).
void ensure_engine_basis(Solver& S, int engine) {
  const Problem& p = S.p;
  auto up = [&](DBuf<float>& d, const std::vector<float>& h) {
    d.alloc(h.size());
    CK(cudaMemcpyAsync(d.p, h.data(), d.bytes(), cudaMemcpyHostToDevice, S.stream));
  };
  if (engine == ICNNM_ENGINE_FFMA && !S.Krm.p) {
    std::vector<float> Krm, KT;
    pack_basis(p, S.K.data(), Krm, KT);
    up(S.Krm, Krm);
    up(S.KT, KT);
    CK(cudaStreamSynchronize(S.stream));
  }
  const bool f16 = engine == ICNNM_ENGINE_F16X3;
  if ((engine == ICNNM_ENGINE_TF32X3 || (f16 && f16_debug_mask())) && !S.BpkF.p) {
    up(S.BpkF, pack_b_tiles(p, S.tp, S.K.data(), true));
    up(S.BpkA, pack_b_tiles(p, S.tp, S.K.data(), false));
    CK(cudaStreamSynchronize(S.stream));
  }
  if (f16 && !S.BpkF16.p) {
    // packed on the device (host packing cost ~9 ms per call at k = 405)
    f16_basis_scale(p, S.tp16, S.K.data());
    DBuf<double> dK(static_cast<size_t>(p.k) * p.k);
    CK(cudaMemcpyAsync(dK.p, S.K.data(), dK.bytes(), cudaMemcpyHostToDevice, S.stream));
    pack_b_tiles_f16_device(p, S.tp16, dK.p, true, S.BpkF16, S.stream);
    pack_b_tiles_f16_device(p, S.tp16, dK.p, false, S.BpkA16, S.stream);
    CK(cudaStreamSynchronize(S.stream));
  }
}

// Programmatic dependent launch for the kernel-to-kernel edges of the
// iteration graph (adjoint <- coef, update <- adjoint, forward <- update):
// the successor's prologue overlaps its predecessor's tail.  Off for the
// sharded solve (copies / NCCL between the kernels), the per-family profile
// and ICNNM_PDL=0.
bool use_pdl(const Solver& S) {
  static const bool on = env_knob("ICNNM_PDL", 1) != 0;
  return on && !S.sharded && !S.profile;
}

void launch_fwd(Solver& S, Slab& s, int mode) {
  // mode 2 (exact residual): forward on L_{t+1}, epilogue sums the gap into slot[5]
  const float* src = mode == 2 ? s.Lr.p : s.Lt.p;
  double* acc = mode == 2 ? S.red.p + engine_kp(S) + 5 : S.red.p;
  if (is_tc(S.engine)) {
    const bool f16 = S.engine == ICNNM_ENGINE_F16X3 && !(f16_debug_mask() & 2);
    double* part = nullptr;
    if (S.det) {
      const size_t row0 = static_cast<size_t>(slab_index(S, s)) * S.nsm;
      part = mode == 2 ? S.gpart.p + row0 : S.npart.p + row0 * engine_kp(S);
    }
    launch_tc_kernel(s.gtc, f16 ? S.tp16 : S.tp, true, mode, src, s.W.p,
                     f16 ? S.BpkF16.p : S.BpkF.p, S.cvec.p, s.adj.p, acc, S.st.p, S.stream,
                     S.tc_counters ? S.dbg.p : nullptr, 0.f, mode != 0 && use_pdl(S), nullptr,
                     part);
    ++S.launches;
    return;
  }
  icnnm_dev::icnnm_fwd_ffma<<<static_cast<unsigned>(n_bricks(s.g)), 128, fwd_smem(s.g),
                              S.stream>>>(s.g, src, S.Krm.p, s.W.p, S.cvec.p, S.st.p, acc, mode);
  CKL();
  ++S.launches;
}
void launch_adj(Solver& S, Slab& s) {
  if (is_tc(S.engine)) {
    const bool f16 = S.engine == ICNNM_ENGINE_F16X3 && !(f16_debug_mask() & 1);
    launch_tc_kernel(s.gtc, f16 ? S.tp16 : S.tp, false, 1, s.Lt.p, s.W.p,
                     f16 ? S.BpkA16.p : S.BpkA.p, S.cvec.p, s.adj.p, S.red.p, S.st.p, S.stream,
                     S.tc_counters ? S.dbg.p + icnnm_dev::tc::DBG_SLOTS : nullptr, 0.f,
                     use_pdl(S), S.det ? s.adjq.p : nullptr);
    ++S.launches;
    if (S.det && S.sharded) {
      // {hi, lo} pairs -> adj (fp32), accumulator cleared for the next launch
      // (sharded: the halo rows of adj are exchanged before the update; the
      // unsharded update folds the pairs itself, launch_update)
      const int64_t n = static_cast<int64_t>(s.gtc.Hsrc) * s.gtc.W * s.gtc.T;
      cudaLaunchConfig_t lc{};
      cudaLaunchAttribute at{};
      at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at.val.programmaticStreamSerializationAllowed = 1;
      lc.gridDim = dim3(static_cast<unsigned>((n + 255) / 256));
      lc.blockDim = dim3(256);
      lc.stream = S.stream;
      lc.attrs = &at;
      lc.numAttrs = use_pdl(S) ? 1 : 0;
      CK(cudaLaunchKernelEx(&lc, icnnm_dev::icnnm_adj_q2f, n,
                            static_cast<const icnnm_dev::IterState*>(S.st.p), s.adjq.p, s.adj.p));
      ++S.launches;
    }
    return;
  }
  icnnm_dev::icnnm_adj_ffma<<<static_cast<unsigned>(n_bricks(s.g)), 128, adj_smem(s.g),
                              S.stream>>>(s.g, s.W.p, S.KT.p, S.cvec.p, s.adj.p, S.st.p, 1);
  CKL();
  ++S.launches;
}

int engine_kp(const Solver& S) {
  return is_tc(S.engine) ? S.tp.kp : S.p.kp;
}

// The iteration's partial rows for the fold (or none in the atomic mode).
icnnm_dev::Partials partials(const Solver& S) {
  icnnm_dev::Partials P{};
  if (!S.det) return P;
  const int ns = static_cast<int>(S.slabs.size());
  P.npart = S.npart.p;
  P.nrows = ns * S.nsm;
  P.upart = S.upart.p;
  P.urows = ns * S.upd_rows;
  if (S.exact_res) {
    P.gpart = S.gpart.p;
    P.grows = ns * S.nsm;
  }
  return P;
}

// Deterministic buffers of a tcgen05 run, allocated before any graph capture.
void prepare_det(Solver& S) {
  // ICNNM_DET=0 (experiments build): fp32 / fp64 atomics instead (A/B)
  static const int det_env = env_knob("ICNNM_DET", 1);
  S.det = is_tc(S.engine) && det_env != 0;
  if (!S.det) return;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&S.nsm, cudaDevAttrMultiProcessorCount, dev));
  S.upd_rows = 0;
  for (auto& s : S.slabs) S.upd_rows = std::max(S.upd_rows, update_grid(s.m_own));
  const int ns = static_cast<int>(S.slabs.size());
  const int kpe = engine_kp(S);
  const bool f16 = S.engine == ICNNM_ENGINE_F16X3;
  const TcPlan& t = f16 ? S.tp16 : S.tp;
  const size_t nrow = static_cast<size_t>(ns) * S.nsm;
  auto zero = [&](DBuf<double>& b, size_t n) {
    if (b.n != n) {
      b.alloc(n);
      CK(cudaMemsetAsync(b.p, 0, b.bytes(), S.stream));
    }
  };
  zero(S.npart, nrow * kpe);
  zero(S.gpart, nrow);
  zero(S.upart, static_cast<size_t>(ns) * S.upd_rows * 8);
  (void)t;
  for (auto& s : S.slabs) {
    const size_t need = static_cast<size_t>(s.gtc.Hsrc) * s.gtc.W * s.gtc.T;
    if (s.adjq.n != need) {
      s.adjq.alloc(need);
      CK(cudaMemsetAsync(s.adjq.p, 0, s.adjq.bytes(), S.stream));
    }
  }
}

void launch_coef(Solver& S, const icnnm_solver_config& cfg, double kd, double res_scale,
                 double floor_rel) {
  // sharded solves fold before the all-reduce (icnnm_fold); else the coef
  // kernel folds
  const icnnm_dev::Partials P = S.sharded ? icnnm_dev::Partials{} : partials(S);
  // work-skipping timing experiments (experiments build): garbage iterates stop
  // changing, which would end the solve on l_change = 0
  static const bool never_stop = env_knob("ICNNM_NEVER_STOP", 0) != 0;
  icnnm_dev::icnnm_coef<<<1, 1024, 0, S.stream>>>(S.st.p, S.theta.p, S.red.p, S.cvec.p,
                                                  S.stats.p, S.p.k, engine_kp(S), kd, res_scale,
                                                  cfg.tol_primal, never_stop ? -1.0 : cfg.tol_change,
                                                  floor_rel, S.exact_res ? 1 : 0, P);
  CKL();
}

void launch_update(Solver& S, Slab& s, const icnnm_solver_config& cfg, double kd, bool pdl) {
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute at{};
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  lc.gridDim = dim3(update_grid(s.m_own));
  lc.blockDim = dim3(256);
  lc.stream = S.stream;
  lc.attrs = &at;
  lc.numAttrs = pdl ? 1 : 0;
  double* upart =
      S.det ? S.upart.p + static_cast<size_t>(slab_index(S, s)) * S.upd_rows * 8 : nullptr;
  CK(cudaLaunchKernelEx(&lc, icnnm_dev::icnnm_update, s.m_own,
                        static_cast<const icnnm_dev::IterState*>(S.st.p), cfg.lambda, kd,
                        s.adj.p + s.halo_elems, s.L.p, s.V.p, static_cast<const float*>(s.pm.p),
                        static_cast<const float*>(s.mask.p), s.Lt.p + s.halo_elems,
                        S.red.p + engine_kp(S),
                        S.exact_res ? s.Lr.p + s.halo_elems : static_cast<float*>(nullptr),
                        upart,
                        (S.det && !S.sharded && is_tc(S.engine)) ? s.adjq.p
                                                                 : static_cast<float2*>(nullptr)));
}

void allreduce_red(Solver& S) {
  if (S.sharded && S.det) {
    // fold the slabs' partial rows into red before the cross-rank sum
    icnnm_dev::icnnm_fold<<<1, 1024, 0, S.stream>>>(partials(S), engine_kp(S), S.red.p);
    CKL();
    ++S.launches;
  }
  if (S.comm) S.comm->allreduce_sum(S.red.p, engine_kp(S) + 8, S.stream);
}

struct RunResult {
  std::vector<IterStats> stats;
  IterState st{};
  double loop_ms = 0;
  double run_ms = 0;
};

// One full solve of the staged problem (device-resident hot path).
RunResult solver_run_f64(Solver& S, const icnnm_solver_config& cfg);

RunResult solver_run(Solver& S, const icnnm_solver_config& cfg_in) {
  if (!S.uploaded) invalid("solve: no problem uploaded");
  const icnnm_solver_config cfg = resolve_engine(cfg_in);
  if (cfg.engine == ICNNM_ENGINE_F64) return solver_run_f64(S, cfg);
  const Problem& p = S.p;
  S.engine = cfg.engine;
  ensure_engine_basis(S, S.engine);
  S.exact_res = cfg.exact_residual != 0;
  prepare_det(S);
  if (S.exact_res)
    for (auto& s : S.slabs)
      if (!s.Lr.p) s.Lr.alloc(s.Lt.n);
  const int iters = cfg.max_iters;
  const double kd = static_cast<double>(p.k);
  // theta schedule exactly as solver.cpp:88-91,126 (fp64, sequential).
  std::vector<double> th(iters + 1);
  double t0 = cfg.has_theta0 ? cfg.theta0 : 1e-2 * S.pm_absmax * kd;
  if (t0 <= 0) t0 = 1e-2;
  t0 = std::min(t0, cfg.theta_max);
  th[0] = t0;
  for (int i = 1; i <= iters; ++i) th[i] = std::min(th[i - 1] * cfg.theta_growth, cfg.theta_max);
  double res_scale = std::sqrt(kd) * std::sqrt(S.pm_norm2);
  if (res_scale == 0) res_scale = 1.0;
  const double mean = S.pm_sum / static_cast<double>(S.observed);

  S.theta.alloc(iters + 1);
  S.stats.alloc(iters);
  // One ADMM iteration as a graph: coef -> adjoint -> update -> forward.
  const double floor_rel = 1e-5;
  auto iteration = [&]() {
    launch_coef(S, cfg, kd, res_scale, floor_rel);
    for (auto& s : S.slabs) launch_adj(S, s);
    exchange_adj(S);
    for (auto& s : S.slabs) launch_update(S, s, cfg, kd, use_pdl(S));
    exchange_lt(S);
    if (S.exact_res) {
      exchange_lt(S, &Slab::Lr);
      for (auto& s : S.slabs) launch_fwd(S, s, 2);
    }
    for (auto& s : S.slabs) launch_fwd(S, s, 1);
    allreduce_red(S);
  };


  if (S.tc_counters && !S.dbg.p) S.dbg.alloc(2 * icnnm_dev::tc::DBG_SLOTS);  // captured pointer
  // pinned staging of the per-run host inputs (theta schedule, initial state),
  // so that their uploads are capturable stream operations
  // pinned staging from a grow-only per-thread pool (cudaMallocHost per call
  // occasionally cost tens of ms in the end-to-end path); run() completes the
  // solve before returning, so solvers on one thread never share it in flight
  struct PinnedPool {
    void* p = nullptr;
    size_t bytes = 0;
    ~PinnedPool() {
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local PinnedPool pool;
  const size_t need = 2 * sizeof(IterState) + th.size() * sizeof(double);
  if (pool.bytes < need) {
    if (pool.p) cudaFreeHost(pool.p);
    pool.p = nullptr;
    pool.bytes = 0;
    const size_t want = std::max<size_t>(need, 64 * 1024);
    CK(cudaMallocHost(&pool.p, want));
    pool.bytes = want;
  }
  S.h_st = static_cast<IterState*>(pool.p);
  S.h_theta = reinterpret_cast<double*>(static_cast<char*>(pool.p) + 2 * sizeof(IterState));
  std::copy(th.begin(), th.end(), S.h_theta);
  IterState st0{};
  st0.active = 1;
  st0.max_iters = iters;
  S.h_st[0] = st0;

  // setup of one solve: theta/state upload, L0 = pm (or mean fill), W = A(L0)K
  const int64_t WT = p.dims[1] * p.dims[2];
  // events may be recorded inside a stream capture: "external" records become
  // event-record nodes of the graph (a plain record would only add an edge)
  auto record = [&](cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(S.stream, &cs));
    if (cs == cudaStreamCaptureStatusActive)
      CK(cudaEventRecordWithFlags(e, S.stream, cudaEventRecordExternal));
    else
      CK(cudaEventRecord(e, S.stream));
  };
  auto setup = [&]() {
    record(S.evs);
    CK(cudaMemcpyAsync(S.theta.p, S.h_theta, th.size() * sizeof(double), cudaMemcpyHostToDevice,
                       S.stream));
    CK(cudaMemsetAsync(S.stats.p, 0, S.stats.bytes(), S.stream));
    CK(cudaMemsetAsync(S.red.p, 0, S.red.bytes(), S.stream));
    CK(cudaMemcpyAsync(S.st.p, S.h_st, sizeof(IterState), cudaMemcpyHostToDevice, S.stream));
    if (S.tc_counters) CK(cudaMemsetAsync(S.dbg.p, 0, S.dbg.bytes(), S.stream));
    for (auto& s : S.slabs) {
      const int64_t off = (s.row0 - S.slabs[0].row0) * WT;
      icnnm_dev::icnnm_setup<<<grid_for(s.m_own, 256), 256, 0, S.stream>>>(
          s.m_own, S.Mstage.p + off, S.maskstage.p + off, cfg.init_fill == ICNNM_INIT_MEAN,
          mean, s.pm.p, s.mask.p, s.L.p, s.V.p, s.Lt.p + s.halo_elems);
      CKL();
      ++S.launches;
      CK(cudaMemsetAsync(s.W.p, 0, s.W.bytes(), S.stream));
      CK(cudaMemsetAsync(s.adj.p, 0, s.adj.bytes(), S.stream));
      if (s.adjq.p) CK(cudaMemsetAsync(s.adjq.p, 0, s.adjq.bytes(), S.stream));
    }
    exchange_lt(S);
    for (auto& s : S.slabs) launch_fwd(S, s, 0);
    allreduce_red(S);
  };
  // final coef: moves the last update slot into stats, evaluates the stop test.
  auto finish = [&]() {
    launch_coef(S, cfg, kd, res_scale, floor_rel);
    ++S.launches;
    record(S.ev1);
  };

  S.launches = 0;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};  // destroyed after the final sync
  if (S.profile) {
    setup();
    CK(cudaEventRecord(S.ev0, S.stream));
    // Per-family timing (serialised, events between launches; diagnostics).
    cudaEvent_t e[5];
    for (auto& x : e) CK(cudaEventCreate(&x));
    double acc[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
      CK(cudaEventRecord(e[0], S.stream));
      launch_coef(S, cfg, kd, res_scale, floor_rel);
      CK(cudaEventRecord(e[1], S.stream));
      for (auto& s : S.slabs) launch_adj(S, s);
      exchange_adj(S);
      CK(cudaEventRecord(e[2], S.stream));
      for (auto& s : S.slabs) launch_update(S, s, cfg, kd, false);
      exchange_lt(S);
      if (S.exact_res) {
        exchange_lt(S, &Slab::Lr);
        for (auto& s : S.slabs) launch_fwd(S, s, 2);
      }
      CK(cudaEventRecord(e[3], S.stream));
      for (auto& s : S.slabs) launch_fwd(S, s, 1);
      allreduce_red(S);
      CK(cudaEventRecord(e[4], S.stream));
      CK(cudaEventSynchronize(e[4]));
      float ms;
      CK(cudaEventElapsedTime(&ms, e[0], e[1])); acc[3] += ms;
      CK(cudaEventElapsedTime(&ms, e[1], e[2])); acc[1] += ms;
      CK(cudaEventElapsedTime(&ms, e[2], e[3])); acc[2] += ms;
      if (it < iters - 1) { CK(cudaEventElapsedTime(&ms, e[3], e[4])); acc[0] += ms; }
    }
    S.prof_ms[0] = iters > 1 ? acc[0] / (iters - 1) : 0;
    S.prof_ms[1] = acc[1] / iters;
    S.prof_ms[2] = acc[2] / iters;
    S.prof_ms[3] = acc[3] / iters;
    for (auto& x : e) cudaEventDestroy(x);
    finish();
  } else {
    // The solve -- setup, its events, every iteration, the final coef -- runs as
    // CUDA graphs captured and instantiated before they are launched, so the
    // device time of a solve can never be stretched by host-side delays
    // inside a graph.  A long solve is split: a head graph (setup + H
    // iterations) is launched first, and the rest is captured and
    // instantiated while the head runs on the device (capture+instantiate
    // costs ~30 us per iteration on the host: 8-9 ms of every end-to-end call
    // at config 2 otherwise).  H is sized from the contraction's flops so the
    // head outlasts that capture 3x over; short or small solves stay one graph.
    // Solves longer than GMAX replay a GMAX-iteration body graph; replays past
    // max_iters are no-ops (the coef kernel deactivates), and with tolerances
    // the host checks the state between replays.
    constexpr int GMAX = 512;
    const bool may_stop = !(cfg.tol_primal <= 1e-200 && cfg.tol_change <= 1e-200);
    const double t_it = 4.0 * static_cast<double>(p.m) * kd * kd / 2.0e14 + 25e-6;  // s, est.
    const double cap_it = 30e-6;                                                      // s, host
    int H = iters;
    if (S.graph_split && iters > 1) {
      const double need = 3.0 * (cap_it * std::min(iters, GMAX) + 2e-3);
      const int h = static_cast<int>(std::ceil(need / t_it));
      if (2 * h <= iters) H = std::max(h, 1);
    }
    if (H > GMAX) H = GMAX;
    const bool one = H == iters;  // head graph holds the whole solve, final coef included
    auto capture = [&](bool head, int n, bool tail) {
      cudaGraph_t g = nullptr;
      cudaGraphExec_t e = nullptr;
      CK(cudaStreamBeginCapture(S.stream, cudaStreamCaptureModeThreadLocal));
      if (head) {
        setup();
        record(S.ev0);
      }
      for (int u = 0; u < n; ++u) iteration();
      if (tail) finish();
      CK(cudaStreamEndCapture(S.stream, &g));
      CK(cudaGraphInstantiate(&e, g, 0));
      CK(cudaGraphUpload(e, S.stream));
      cudaGraphDestroy(g);
      return e;
    };
    // launch accounting: capture counts the TC/FFMA launches of one iteration
    const int64_t l0 = S.launches;
    g_timer.mark("run: schedule/staging");
    cudaGraphExec_t gx = capture(true, H, one);
    g_timer.mark("run: capture+instantiate (head)");
    const int64_t captured = S.launches - l0;
    S.launches = l0;
    // per iteration: coef + update per slab + the counted engine launches
    const int64_t setup_l = static_cast<int64_t>(S.slabs.size()) * 2 + (one ? 1 : 0);
    const int64_t per_iter = (captured - setup_l) / std::max(1, H) + 1 +
                             static_cast<int64_t>(S.slabs.size());
    CK(cudaStreamSynchronize(S.stream));  // uploads done; nothing of this solve has run
    g_timer.mark("run: graph upload");
    CK(cudaGraphLaunch(gx, S.stream));
    S.launches += setup_l + per_iter * H;
    cudaGraphExec_t gr = nullptr;
    bool finished = one;
    if (!one) {
      const int R = iters - H;
      const int U = std::min(R, GMAX);
      const bool tail_in = R <= GMAX && !may_stop;  // launched exactly once
      const int64_t l1 = S.launches;
      gr = capture(false, U, tail_in);  // overlaps the head on the device
      S.launches = l1;
      g_timer.mark("run: capture+instantiate (body, overlapped)");
      for (int it = H; it < iters; it += U) {
        if (may_stop) {
          CK(cudaMemcpyAsync(S.h_st + 1, S.st.p, sizeof(IterState), cudaMemcpyDeviceToHost,
                             S.stream));
          CK(cudaStreamSynchronize(S.stream));
          if (!S.h_st[1].active) break;
        }
        CK(cudaGraphLaunch(gr, S.stream));
        S.launches += per_iter * std::min(U, iters - it);
        if (tail_in) {
          finished = true;
          S.launches += 1;
        }
      }
    }
    if (!finished) finish();
    gexec[0] = gx;
    gexec[1] = gr;
  }
  RunResult R;
  R.stats.resize(iters);
  CK(cudaMemcpyAsync(R.stats.data(), S.stats.p, S.stats.bytes(), cudaMemcpyDeviceToHost,
                     S.stream));
  CK(cudaMemcpyAsync(&R.st, S.st.p, sizeof(IterState), cudaMemcpyDeviceToHost, S.stream));
  CK(cudaStreamSynchronize(S.stream));
  g_timer.mark("run: device solve");
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, S.ev0, S.ev1));
  R.loop_ms = ms;
  CK(cudaEventElapsedTime(&ms, S.evs, S.ev1));
  R.run_ms = ms;
  for (auto& x : gexec)
    if (x) cudaGraphExecDestroy(x);
  return R;
}

// Report of solver.cpp:128-139 from the device statistics.
// ICNNM_ENGINE_F64: the literal fp64 loop (icnnm_cnnm.cu) on the staged problem.
RunResult solver_run_f64(Solver& S, const icnnm_solver_config& cfg) {
  if (S.sharded) invalid("solve: the fp64 engine does not run H-sharded solves");
  RunResult R;
  S.engine = ICNNM_ENGINE_F64;
  S.exact_res = true;  // the report's residual is the exact gap norm
  S.launches = 0;
  CK(cudaStreamSynchronize(S.stream));  // the staged problem is on the device
  int iters = 0, conv = 0;
  double ms = 0;
  Slab& s = S.slabs[0];
  icnnm_f64_loop(S.p, S.Mstage.p, S.maskstage.p, S.K.data(), cfg, S.pm_absmax, S.pm_norm2,
                 S.pm_sum, S.observed, s.L.p, R.stats, &iters, &conv, &ms);
  R.st.next_it = iters;
  R.st.it = iters - 1;
  R.st.converged = conv;
  R.st.active = 0;
  R.st.max_iters = cfg.max_iters;
  R.loop_ms = ms;
  R.run_ms = ms;
  return R;
}

void fill_report(const Solver& S, const icnnm_solver_config& cfg, const RunResult& R,
                 icnnm_solve_report* rep, double wall_s) {
  if (!rep) return;
  const double kd = static_cast<double>(S.p.k);
  double res_scale = std::sqrt(kd) * std::sqrt(S.pm_norm2);
  if (res_scale == 0) res_scale = 1.0;
  const int executed = R.st.next_it;
  int n = 0;
  int term = ICNNM_TERM_MAX_ITERS;
  for (int it = 0; it < executed; ++it) {
    const IterStats& q = R.stats[it];
    const double gap2 = S.exact_res ? q.gap2 : q.z2 - 2.0 * q.ip + kd * q.ln2;
    const double res = std::sqrt(std::max(gap2, 0.0)) / res_scale;
    const bool res_ok = S.exact_res || gap2 > 1e-5 * (q.z2 + kd * q.ln2);
    const double lc = std::sqrt(q.dl2) / std::max(std::sqrt(q.l2o), 1e-300);
    if (rep->objective) rep->objective[it] = q.l21 + 0.5 * cfg.lambda * kd * q.fit;
    // Below the fp32 floor the identity cannot resolve the gap: report NaN
    // (never "converged" on it) instead of a rounding artefact.
    if (rep->primal_residual) rep->primal_residual[it] = res_ok ? res : std::nan("");
    if (rep->l_change) rep->l_change[it] = lc;
    n = it + 1;
    if ((res_ok && res < cfg.tol_primal) || lc < cfg.tol_change) {
      term = ICNNM_TERM_CONVERGED;
      break;
    }
  }
  rep->iterations = n;
  rep->termination = term;
  rep->wall_time_seconds = wall_s;
  rep->loop_seconds = R.loop_ms * 1e-3;
  rep->device_seconds = R.run_ms * 1e-3;
}

void solver_download(Solver& S, double* L_out) {
  if (!L_out) invalid("null output");
  int64_t off = 0;
  for (auto& s : S.slabs) {
    CK(cudaMemcpyAsync(L_out + off, s.L.p, s.m_own * sizeof(double), cudaMemcpyDeviceToHost,
                       S.stream));
    off += s.m_own;
  }
  CK(cudaStreamSynchronize(S.stream));
}

}  // namespace icnnm_host

using namespace icnnm_host;

struct icnnm_solver_s {
  Solver S;
};

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

void icnnm_default_config(icnnm_solver_config* c) {
  if (!c) return;
  c->lambda = 1000.0;
  c->has_theta0 = 0;
  c->theta0 = 0.0;
  c->theta_growth = 1.05;
  c->theta_max = 1e10;
  c->max_iters = 1000;
  c->tol_primal = 1e-7;
  c->tol_change = 1e-8;
  c->rank_tol = 1e-8;
  c->init_fill = ICNNM_INIT_ZERO;
  c->engine = ICNNM_ENGINE_AUTO;
  c->exact_residual = 0;
}

int icnnm_validate_config(const icnnm_solver_config* cfg) {
  return guard([&] { validate_cfg(cfg); });
}

const char* icnnm_last_error(void) { return g_last_error.c_str(); }

int icnnm_empty_cache(void) {
  return guard([&] { devcache_empty(); });
}

const char* icnnm_version(void) { return "icnnm_b200 0.1 (sm_100a)"; }

int icnnm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int icnnm_solver_create(int order, const int64_t* dims, const int64_t* kdims,
                        const double* K_colmajor, const double* eigenvalues, int device,
                        icnnm_solver_t* out) {
  return guard([&] {
    if (!out) invalid("null handle pointer");
    *out = nullptr;
    Problem p = make_problem(order, dims, kdims);
    validate_basis(p.k, K_colmajor, eigenvalues);
    DeviceScope ds(device);
    auto h = std::make_unique<icnnm_solver_s>();
    Solver& S = h->S;
    S.p = p;
    S.device = device;
    S.K.assign(K_colmajor, K_colmajor + static_cast<size_t>(p.k) * p.k);
    S.slabs.resize(1);
    S.slabs[0].row0 = 0;
    S.slabs[0].rows = p.dims[0];
    solver_alloc(S);
    *out = h.release();
  });
}

int icnnm_solver_upload(icnnm_solver_t h, const double* M, const double* mask) {
  return guard([&] {
    if (!h) invalid("null handle");
    DeviceScope ds(h->S.device);
    solver_upload(h->S, M, mask);
  });
}

int icnnm_solver_run(icnnm_solver_t h, const icnnm_solver_config* cfg,
                     icnnm_solve_report* report) {
  return guard([&] {
    if (!h) invalid("null handle");
    validate_cfg(cfg);
    DeviceScope ds(h->S.device);
    g_timer.reset();
    auto t0 = std::chrono::steady_clock::now();
    RunResult R = solver_run(h->S, *cfg);
    double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fill_report(h->S, *cfg, R, report, wall);
  });
}

int icnnm_solver_download(icnnm_solver_t h, double* L_out) {
  return guard([&] {
    if (!h) invalid("null handle");
    DeviceScope ds(h->S.device);
    solver_download(h->S, L_out);
  });
}

int64_t icnnm_solver_last_launches(icnnm_solver_t h) { return h ? h->S.launches : -1; }

int64_t icnnm_solver_device_bytes(icnnm_solver_t h) {
  if (!h) return -1;
  const Solver& S = h->S;
  int64_t b = S.Krm.bytes() + S.KT.bytes() + S.cvec.bytes() + S.red.bytes() + S.theta.bytes() +
              S.stats.bytes() + S.Mstage.bytes() + S.maskstage.bytes();
  for (auto& s : S.slabs)
    b += s.Lt.bytes() + s.adj.bytes() + s.pm.bytes() + s.mask.bytes() + s.W.bytes() +
         s.L.bytes() + s.V.bytes();
  return b;
}

int icnnm_solver_set_profile(icnnm_solver_t h, int enable) {
  return guard([&] {
    if (!h) invalid("null handle");
    h->S.profile = (enable & 1) != 0;
    h->S.tc_counters = (enable & 2) != 0;
  });
}

int icnnm_solver_tc_counters(icnnm_solver_t h, unsigned long long* out) {  // 2 x DBG_SLOTS
  return guard([&] {
    if (!h || !out) invalid("null argument");
    const int n = 2 * icnnm_dev::tc::DBG_SLOTS;
    if (!h->S.dbg.p) {
      for (int i = 0; i < n; ++i) out[i] = 0;
      return;
    }
    DeviceScope ds(h->S.device);
    CK(cudaMemcpy(out, h->S.dbg.p, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

int icnnm_solver_kernel_times(icnnm_solver_t h, double* out) {
  return guard([&] {
    if (!h || !out) invalid("null argument");
    for (int i = 0; i < 4; ++i) out[i] = h->S.prof_ms[i];
  });
}

void icnnm_solver_destroy(icnnm_solver_t h) {
  if (!h) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(h->S.device);
  delete h;
  if (prev >= 0) cudaSetDevice(prev);
}

int icnnm_cuda_solve(int order, const int64_t* dims, const double* M_obs, const double* mask,
                     const int64_t* kdims, const double* K_colmajor, const double* eigenvalues,
                     const icnnm_solver_config* cfg, int device, double* L_out,
                     icnnm_solve_report* report) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    g_timer.reset();
    validate_cfg(cfg);
    Problem p = make_problem(order, dims, kdims);
    if (!L_out) invalid("null output");
    validate_basis(p.k, K_colmajor, eigenvalues);
    g_timer.mark("validate basis");
    DeviceScope ds(device);
    {
      Solver S;
      S.p = p;
      S.device = device;
      S.K.assign(K_colmajor, K_colmajor + static_cast<size_t>(p.k) * p.k);
      S.slabs.resize(1);
      S.slabs[0].rows = p.dims[0];
      solver_alloc(S);
      solver_upload(S, M_obs, mask);
      g_timer.mark("upload (validate+H2D)");
      RunResult R = solver_run(S, *cfg);
      solver_download(S, L_out);
      g_timer.mark("download");
      double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      fill_report(S, *cfg, R, report, wall);
    }
    g_timer.mark("release");
  });
}

int icnnm_cuda_solve_batch(int n, int order, const int64_t* dims, const double* const* M_obs,
                           const double* const* masks, const int64_t* kdims,
                           const double* K_colmajor, const double* eigenvalues,
                           const icnnm_solver_config* cfg, const int* devices, int n_devices,
                           double* const* L_out, icnnm_solve_report* reports) {
  return guard([&] {
    if (n < 0) invalid("solve_batch: negative batch size");
    if (n == 0) return;
    if (!M_obs || !masks || !L_out) invalid("solve_batch: null input/output array");
    if (!devices || n_devices < 1) invalid("solve_batch: no devices");
    validate_cfg(cfg);
    Problem p = make_problem(order, dims, kdims);
    for (int i = 0; i < n; ++i)
      if (!M_obs[i] || !masks[i] || !L_out[i])
        invalid("solve_batch: null tensor pointer at index " + std::to_string(i));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    for (int d = 0; d < n_devices; ++d)
      if (devices[d] < 0 || devices[d] >= ndev)
        invalid("device index " + std::to_string(devices[d]) + " out of range (" +
                std::to_string(ndev) + " devices)");
    validate_basis(p.k, K_colmajor, eigenvalues);  // once: one shared basis
    // contiguous blocks of problems per device; one worker thread per device
    const int nw = std::min(n, n_devices);
    struct Outcome {
      int code = ICNNM_OK;
      int index = -1;
      std::string msg;
    };
    std::vector<Outcome> out(nw);
    auto worker = [&](int w) {
      const int i0 = static_cast<int>(static_cast<int64_t>(n) * w / nw);
      const int i1 = static_cast<int>(static_cast<int64_t>(n) * (w + 1) / nw);
      int cur = i0;
      const int rc = guard([&] {
        DeviceScope ds(devices[w]);
        Solver S;
        S.p = p;
        S.device = devices[w];
        S.K.assign(K_colmajor, K_colmajor + static_cast<size_t>(p.k) * p.k);
        S.slabs.resize(1);
        S.slabs[0].rows = p.dims[0];
        solver_alloc(S);
        for (cur = i0; cur < i1; ++cur) {
          const auto t0 = std::chrono::steady_clock::now();
          solver_upload(S, M_obs[cur], masks[cur]);
          RunResult R = solver_run(S, *cfg);
          solver_download(S, L_out[cur]);
          const double wall =
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          if (reports) fill_report(S, *cfg, R, reports + cur, wall);
        }
      });
      if (rc != ICNNM_OK) out[w] = {rc, cur, g_last_error};
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < nw; ++w) pool.emplace_back(worker, w);
    worker(0);
    for (auto& t : pool) t.join();
    for (const Outcome& o : out)
      if (o.code != ICNNM_OK)
        fail(o.code, "solve_batch: problem " + std::to_string(o.index) + ": " + o.msg);
  });
}

// --------------------------------------------------------------------------
// Operator level
// --------------------------------------------------------------------------
int icnnm_cuda_conv_forward_ex(int order, const int64_t* dims, const double* L,
                               const int64_t* kdims, const double* K_colmajor, int engine,
                               int device, double* out) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    if (!L || !K_colmajor || !out) invalid("null argument");
    if (engine != ICNNM_ENGINE_FFMA && !is_tc(engine)) invalid("unknown engine");
    DeviceScope ds(device);
    set_smem_attrs();
    Geo g = make_geo(p, p.dims[0], true);
    const int64_t H = p.dims[0], W = p.dims[1], T = p.dims[2];
    std::vector<float> Lf(L, L + p.m);
    DBuf<float> dL(p.m);
    CK(cudaMemcpy(dL.p, Lf.data(), dL.bytes(), cudaMemcpyHostToDevice));
    if (is_tc(engine)) {
      TcPlan t = tc_plan(p, engine == ICNNM_ENGINE_F16X3);
      Geo gt = tc_geo(g, t);
      t.vmap = gt.vmap;
      check_smem(icnnm_dev::tc::smem_bytes(gt, true, 2, 2, t.f16));
      auto bf = pack_b_tiles(p, t, K_colmajor, true);
      DBuf<float> dB(bf.size()), dW(tc_w_elems(gt, t));
      DBuf<double> dn(t.kp);
      CK(cudaMemcpy(dB.p, bf.data(), dB.bytes(), cudaMemcpyHostToDevice));
      CK(cudaMemset(dn.p, 0, dn.bytes()));
      launch_tc_kernel(gt, t, true, 0, dL.p, dW.p, dB.p, nullptr, nullptr, dn.p, nullptr, 0);
      std::vector<float> Wh(dW.n);
      CK(cudaMemcpy(Wh.data(), dW.p, dW.bytes(), cudaMemcpyDeviceToHost));
      for (int64_t h = 0; h < H; ++h)
        for (int64_t w = 0; w < W; ++w)
          for (int64_t tt = 0; tt < T; ++tt) {
            const int64_t flat = (h * W + w) * T + tt;
            const int64_t r = brick_row(gt, h, w, tt);
            const int64_t b = r / BM, v = r % BM;
            for (int j = 0; j < p.k; ++j)
              out[static_cast<size_t>(j) * p.m + flat] =
                  Wh[(static_cast<size_t>(b) * t.kp + j) * 128 + v];
          }
      return;
    }
    check_smem(fwd_smem(g));
    std::vector<float> Krm, KT;
    pack_basis(p, K_colmajor, Krm, KT);
    DBuf<float> dK(Krm.size()), dW(static_cast<size_t>(n_bricks(g)) * BM * p.kp);
    DBuf<double> dn(p.kp);
    CK(cudaMemcpy(dK.p, Krm.data(), dK.bytes(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dn.p, 0, dn.bytes()));
    icnnm_dev::icnnm_fwd_ffma<<<static_cast<unsigned>(n_bricks(g)), 128, fwd_smem(g)>>>(
        g, dL.p, dK.p, dW.p, nullptr, nullptr, dn.p, 0);
    CKL();
    std::vector<float> Wh(dW.n);
    CK(cudaMemcpy(Wh.data(), dW.p, dW.bytes(), cudaMemcpyDeviceToHost));
    for (int64_t h = 0; h < H; ++h)
      for (int64_t w = 0; w < W; ++w)
        for (int64_t t = 0; t < T; ++t) {
          const int64_t flat = (h * W + w) * T + t;
          const float* row = Wh.data() + brick_row(g, h, w, t) * p.kp;
          for (int j = 0; j < p.k; ++j) out[static_cast<size_t>(j) * p.m + flat] = row[j];
        }
  });
}

int icnnm_cuda_conv_forward(int order, const int64_t* dims, const double* L,
                            const int64_t* kdims, const double* K_colmajor, int device,
                            double* out) {
  return icnnm_cuda_conv_forward_ex(order, dims, L, kdims, K_colmajor, ICNNM_ENGINE_FFMA, device,
                                    out);
}

int icnnm_cuda_conv_adjoint_ex(int order, const int64_t* dims, const int64_t* kdims,
                               const double* Wcm, int engine, int device, double* out) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    if (!Wcm || !out) invalid("null argument");
    if (engine != ICNNM_ENGINE_FFMA && !is_tc(engine)) invalid("unknown engine");
    DeviceScope ds(device);
    set_smem_attrs();
    Geo g = make_geo(p, p.dims[0], true);
    const int64_t H = p.dims[0], Wd = p.dims[1], T = p.dims[2];
    DBuf<float> dadj(p.m);
    CK(cudaMemset(dadj.p, 0, dadj.bytes()));
    if (is_tc(engine)) {
      TcPlan t = tc_plan(p, engine == ICNNM_ENGINE_F16X3);
      Geo gt = tc_geo(g, t);
      t.vmap = gt.vmap;
      check_smem(icnnm_dev::tc::smem_bytes(gt, false, 2, 2, t.f16));
      std::vector<double> I(static_cast<size_t>(p.k) * p.k, 0.0);
      for (int j = 0; j < p.k; ++j) I[static_cast<size_t>(j) * p.k + j] = 1.0;
      auto ba = pack_b_tiles(p, t, I.data(), false);
      std::vector<float> Wt(tc_w_elems(gt, t), 0.f);
      float wmax = 0.f;  // F16x3 operand scale bound (mode 0: no shrink factors)
      for (int64_t h = 0; h < H; ++h)
        for (int64_t w = 0; w < Wd; ++w)
          for (int64_t tt = 0; tt < T; ++tt) {
            const int64_t flat = (h * Wd + w) * T + tt;
            const int64_t r = brick_row(gt, h, w, tt);
            const int64_t b = r / BM, v = r % BM;
            for (int j = 0; j < p.k; ++j)
            {
              const float x = static_cast<float>(Wcm[static_cast<size_t>(j) * p.m + flat]);
              Wt[(static_cast<size_t>(b) * t.kp + j) * 128 + v] = x;
              wmax = std::max(wmax, std::fabs(x));
            }
          }
      DBuf<float> dB(ba.size()), dW(Wt.size());
      CK(cudaMemcpy(dB.p, ba.data(), dB.bytes(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dW.p, Wt.data(), dW.bytes(), cudaMemcpyHostToDevice));
      launch_tc_kernel(gt, t, false, 0, nullptr, dW.p, dB.p, nullptr, dadj.p, nullptr, nullptr, 0,
                       nullptr, wmax);
    } else {
      check_smem(adj_smem(g));
      // W (m x k column-major) -> brick-ordered rows; K = I.
      std::vector<float> Wb(static_cast<size_t>(n_bricks(g)) * BM * p.kp, 0.f);
      for (int64_t h = 0; h < H; ++h)
        for (int64_t w = 0; w < Wd; ++w)
          for (int64_t t = 0; t < T; ++t) {
            const int64_t flat = (h * Wd + w) * T + t;
            float* row = Wb.data() + brick_row(g, h, w, t) * p.kp;
            for (int j = 0; j < p.k; ++j)
              row[j] = static_cast<float>(Wcm[static_cast<size_t>(j) * p.m + flat]);
          }
      std::vector<float> I(static_cast<size_t>(p.kp) * p.kp, 0.f);
      for (int j = 0; j < p.k; ++j) I[static_cast<size_t>(j) * p.kp + j] = 1.f;
      DBuf<float> dW(Wb.size()), dI(I.size());
      CK(cudaMemcpy(dW.p, Wb.data(), dW.bytes(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dI.p, I.data(), dI.bytes(), cudaMemcpyHostToDevice));
      icnnm_dev::icnnm_adj_ffma<<<static_cast<unsigned>(n_bricks(g)), 128, adj_smem(g)>>>(
          g, dW.p, dI.p, nullptr, dadj.p, nullptr, 0);
      CKL();
    }
    std::vector<float> a(p.m);
    CK(cudaMemcpy(a.data(), dadj.p, dadj.bytes(), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < p.m; ++i) out[i] = a[i];
  });
}

int icnnm_cuda_conv_adjoint(int order, const int64_t* dims, const int64_t* kdims,
                            const double* Wcm, int device, double* out) {
  return icnnm_cuda_conv_adjoint_ex(order, dims, kdims, Wcm, ICNNM_ENGINE_FFMA, device, out);
}

int icnnm_cuda_prox_l21(int64_t rows, int64_t cols, const double* W, double tau, int device,
                        double* Z) {
  return guard([&] {
    if (tau < 0) invalid("prox_l21: tau must be >= 0");
    if (rows < 0 || cols < 0) invalid("prox_l21: negative shape");
    if (rows == 0 || cols == 0) return;
    if (!W || !Z) invalid("null argument");
    DeviceScope ds(device);
    DBuf<double> dW(rows * cols), dZ(rows * cols), dn(cols);
    CK(cudaMemcpy(dW.p, W, dW.bytes(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dn.p, 0, dn.bytes()));
    icnnm_dev::icnnm_colnorm2<<<static_cast<unsigned>(cols), 256>>>(rows, cols, dW.p, dn.p);
    CKL();
    icnnm_dev::icnnm_colscale<<<grid_for(rows * cols, 256), 256>>>(rows, cols, dW.p, dn.p, tau,
                                                                  dZ.p);
    CKL();
    CK(cudaMemcpy(Z, dZ.p, dZ.bytes(), cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

namespace icnnm_host {

// R lags (fp64) of one tensor, accumulated into dR.
void gram_lags_accumulate(const Problem& p, const double* dX, double* dR, cudaStream_t s) {
  const int H = static_cast<int>(p.dims[0]), W = static_cast<int>(p.dims[1]),
            T = static_cast<int>(p.dims[2]);
  const int kh = static_cast<int>(p.kd[0]), kw = static_cast<int>(p.kd[1]),
            kt = static_cast<int>(p.kd[2]);
  const int nlw = 2 * kw - 1, nlt = 2 * kt - 1;
  const int nl = nlw * nlt;
  void* rt = (nlw <= 256) ? icnnm_dev::gram_lags_rt_ptr(kt) : nullptr;
  if (rt != nullptr) {
    // register-tiled kernel: thread (dw, row), rows = bh x bw voxels of bt frames
    const int rsmax = 256 / nlw;
    int bw = std::min(W, rsmax);
    int bh = std::min(H, std::max(1, rsmax / bw));
    int bt = std::min(T, 64);
    const int cw = std::max(2, 2 * kt - 2);              // frames per step (kernel's CW)
    const int btp = (bt + 2 * cw - 1) / (2 * cw) * (2 * cw);
    // two tiles (the next brick's copies overlap the current brick's lags) within
    // the shared memory of a resident CTA: fewer rows per brick until they fit
    const size_t limit = (kt <= 6 ? 110 : 220) * 1024;
    size_t smem = 0;
    for (;;) {
      const size_t tile = static_cast<size_t>(bh) * bw * (btp + 2) +
                          static_cast<size_t>(bh) * (bw + 2 * (kw - 1)) * ((btp + cw) | 1);
      smem = std::max(2 * tile, static_cast<size_t>(bh) * bw * nl) * sizeof(double);
      if (smem <= limit || (bh == 1 && bw == 1)) break;
      if (bh > 1)
        bh = (bh + 1) / 2;
      else
        bw = (bw + 1) / 2;
    }
    check_smem(smem);
    static std::mutex mu;
    static std::map<void*, size_t> attr;  // opt-in dynamic shared memory per instantiation
    {
      std::lock_guard<std::mutex> lk(mu);
      size_t& cur = attr[rt];
      if (smem > cur) {
        CK(cudaFuncSetAttribute(rt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        cur = smem;
      }
    }
    const int nb = ((H + bh - 1) / bh) * ((W + bw - 1) / bw) * ((T + bt - 1) / bt);
    // one resident wave: kh x grid.y CTAs <= resident CTAs (2 per SM for kt <= 6, else 1)
    int nsm = 148;
    {
      int dev = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    const int resident = nsm * (kt <= 6 ? 2 : 1);
    dim3 grid(kh, std::max(1, std::min(nb, std::max(1, resident / kh))));
    DBuf<double> part(static_cast<size_t>(grid.y) * kh * nl);
    int aH = H, aW = W, aT = T, akw = kw, abh = bh, abw = bw, abt = bt;
    const double* aX = dX;
    double* aR = part.p;
    void* args[] = {&aH, &aW, &aT, &akw, &abh, &abw, &abt, &aX, &aR};
    CK(cudaLaunchKernel(rt, grid, dim3(256), args, smem, s));
    icnnm_dev::icnnm_gram_reduce_sym<<<grid_for(static_cast<int64_t>(kh) * nl, 256), 256, 0, s>>>(
        kh, nl, static_cast<int>(grid.y), part.p, dR);
    CKL();
    CK(cudaStreamSynchronize(s));
    return;
  }
  if (nl > 256 * icnnm_dev::GRAM_LPT_HOST)
    invalid("icnnm_b200: kernel (kw, kt) too large for the Gram kernel");
  int bt = T >= 16 ? 16 : (T >= 8 ? 8 : T);
  int bw = W >= 8 ? 8 : W;
  int bh = H >= 2 ? 2 : 1;
  size_t smem = (static_cast<size_t>(bh) * bw * bt +
                 static_cast<size_t>(bh) * (bw + 2 * (kw - 1)) * (bt + 2 * (kt - 1))) *
                sizeof(double);
  check_smem(smem);
  const int nb = ((H + bh - 1) / bh) * ((W + bw - 1) / bw) * ((T + bt - 1) / bt);
  dim3 grid(2 * kh - 1, std::max(1, std::min(nb, 1184 / (2 * kh - 1) + 1)));
  const int64_t nR = static_cast<int64_t>(2 * kh - 1) * nl;
  DBuf<double> part(static_cast<size_t>(grid.y) * nR);
  icnnm_dev::icnnm_gram_lags<<<grid, 256, smem, s>>>(H, W, T, kh, kw, kt, bh, bw, bt, dX,
                                                     part.p);
  CKL();
  icnnm_dev::icnnm_gram_reduce<<<grid_for(nR, 256), 256, 0, s>>>(nR, static_cast<int>(grid.y),
                                                                 part.p, dR);
  CKL();
  CK(cudaStreamSynchronize(s));
}

// G[s,t] = R[(s - t)] over the kernel box (spectral.cpp:62-79).
void gram_from_lags(const Problem& p, const std::vector<double>& R, double* G) {
  const int kh = static_cast<int>(p.kd[0]), kw = static_cast<int>(p.kd[1]),
            kt = static_cast<int>(p.kd[2]);
  const int k = p.k;
  const int nlw = 2 * kw - 1, nlt = 2 * kt - 1;
  for (int s = 0; s < k; ++s) {
    const int sh = s / (kw * kt), sw = (s / kt) % kw, st = s % kt;
    for (int t = 0; t < k; ++t) {
      const int th = t / (kw * kt), tw = (t / kt) % kw, tt = t % kt;
      const int dh = sh - th + kh - 1, dw = sw - tw + kw - 1, dt = st - tt + kt - 1;
      G[static_cast<size_t>(t) * k + s] = R[(static_cast<size_t>(dh) * nlw + dw) * nlt + dt];
    }
  }
}

}  // namespace icnnm_host


extern "C" {

int icnnm_cuda_conv_gram(int order, const int64_t* dims, const double* L, const int64_t* kdims,
                         int device, double* G) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    if (!L || !G) invalid("null argument");
    DeviceScope ds(device);
    set_smem_attrs();
    const size_t nl = static_cast<size_t>(2 * p.kd[0] - 1) * (2 * p.kd[1] - 1) * (2 * p.kd[2] - 1);
    DBuf<double> dX(p.m), dR(nl);
    CK(cudaMemcpy(dX.p, L, dX.bytes(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dR.p, 0, dR.bytes()));
    gram_lags_accumulate(p, dX.p, dR.p, 0);
    std::vector<double> R(nl);
    CK(cudaMemcpy(R.data(), dR.p, dR.bytes(), cudaMemcpyDeviceToHost));
    gram_from_lags(p, R, G);
  });
}

int icnnm_cuda_learn_basis(int n_refs, int order, const int64_t* dims, const double* const* refs,
                           const int64_t* kdims, int device, double* K_out, double* evals_out,
                           int* degenerate) {
  return guard([&] {
    if (n_refs <= 0 || !refs) invalid("learn_ensemble_basis: empty reference list");
    Problem p = make_problem(order, dims, kdims);
    if (!K_out || !evals_out) invalid("null argument");
    DeviceScope ds(device);
    set_smem_attrs();
    const size_t nl = static_cast<size_t>(2 * p.kd[0] - 1) * (2 * p.kd[1] - 1) * (2 * p.kd[2] - 1);
    DBuf<double> dX(p.m), dR(nl);
    CK(cudaMemset(dR.p, 0, dR.bytes()));
    for (int b = 0; b < n_refs; ++b) {
      if (!refs[b]) invalid("learn_ensemble_basis: null reference");
      CK(cudaMemcpy(dX.p, refs[b], dX.bytes(), cudaMemcpyHostToDevice));
      gram_lags_accumulate(p, dX.p, dR.p, 0);
    }
    std::vector<double> R(nl);
    CK(cudaMemcpy(R.data(), dR.p, dR.bytes(), cudaMemcpyDeviceToHost));
    const int k = p.k;
    std::vector<double> G(static_cast<size_t>(k) * k);
    gram_from_lags(p, R, G.data());
    double gmax = 0;
    for (double v : G) gmax = std::max(gmax, std::fabs(v));
    if (gmax == 0.0) {
      std::fill(K_out, K_out + static_cast<size_t>(k) * k, 0.0);
      for (int i = 0; i < k; ++i) K_out[static_cast<size_t>(i) * k + i] = 1.0;
      std::fill(evals_out, evals_out + k, 0.0);
      if (degenerate) *degenerate = 1;
      return;
    }
    int rc = icnnm_host_symeig_impl(k, G.data(), evals_out, K_out);
    if (rc != 0) fail(ICNNM_RUNTIME_ERROR, "eigensolver did not converge");
    // psd_eig_sorted (spectral.cpp:87-98): clamp >= 0, sign fix, sigma = sqrt.
    for (int i = 0; i < k; ++i) {
      evals_out[i] = std::sqrt(std::max(0.0, evals_out[i]));
      double* col = K_out + static_cast<size_t>(i) * k;
      for (int r = 0; r < k; ++r) {
        if (std::fabs(col[r]) > 1e-12) {
          if (col[r] < 0)
            for (int q = 0; q < k; ++q) col[q] = -col[q];
          break;
        }
      }
    }
    if (degenerate) *degenerate = 0;
  });
}

int icnnm_host_symeig(int n, const double* G, double* evals, double* evecs) {
  return guard([&] {
    if (n < 1 || !G || !evals || !evecs) invalid("symeig: bad arguments");
    if (icnnm_host_symeig_impl(n, G, evals, evecs) != 0)
      fail(ICNNM_RUNTIME_ERROR, "eigensolver did not converge");
  });
}

int icnnm_cuda_objective(int order, const int64_t* dims, const double* L, const double* M,
                         const double* mask, const int64_t* kdims, const double* K, double lambda,
                         int device, double* out) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    if (!L || !M || !mask || !K || !out) invalid("null argument");
    validate_basis(p.k, K, nullptr);
    for (int64_t i = 0; i < p.m; ++i)
      if (mask[i] != 0.0 && mask[i] != 1.0) invalid("SamplingMask: entries must be 0 or 1");
    DeviceScope ds(device);
    set_smem_attrs();
    Geo g = make_geo(p, p.dims[0], true);
    std::vector<float> Krm, KT;
    pack_basis(p, K, Krm, KT);
    std::vector<float> Lf(L, L + p.m);
    DBuf<float> dL(p.m), dK(Krm.size()), dW(static_cast<size_t>(n_bricks(g)) * BM * p.kp);
    DBuf<double> dn(p.kp);
    CK(cudaMemcpy(dL.p, Lf.data(), dL.bytes(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dK.p, Krm.data(), dK.bytes(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dn.p, 0, dn.bytes()));
    icnnm_dev::icnnm_fwd_ffma<<<static_cast<unsigned>(n_bricks(g)), 128, fwd_smem(g)>>>(
        g, dL.p, dK.p, dW.p, nullptr, nullptr, dn.p, 0);
    CKL();
    std::vector<double> n2(p.kp);
    CK(cudaMemcpy(n2.data(), dn.p, dn.bytes(), cudaMemcpyDeviceToHost));
    double col_sum = 0;
    for (int j = 0; j < p.k; ++j) col_sum += std::sqrt(n2[j]);
    double fit = 0;
    for (int64_t i = 0; i < p.m; ++i) {
      const double d = (L[i] - M[i]) * mask[i];
      fit += d * d;
    }
    *out = col_sum + 0.5 * lambda * static_cast<double>(p.k) * fit;
  });
}

// --------------------------------------------------------------------------
// Sharded solve
// --------------------------------------------------------------------------
int icnnm_shard_plan(int64_t H, int G, int64_t kh, int g, int64_t* start, int64_t* count) {
  return guard([&] {
    if (G < 1 || g < 0 || g >= G || H < 1 || kh < 1) invalid("shard plan: bad arguments");
    const int64_t base = H / G, extra = H % G;
    const int64_t s = g * base + std::min<int64_t>(g, extra);
    const int64_t c = base + (g < extra ? 1 : 0);
    if (c < 1 || c < kh - 1) invalid("shard plan: slab thinner than the kernel halo (kh-1 rows)");
    if (start) *start = s;
    if (count) *count = c;
  });
}

int icnnm_dist_unique_id(char* out128) {
  return guard([&] {
    if (!out128) invalid("null argument");
    comm_unique_id(out128);
  });
}

namespace {
// The H-sharded solve of one process: `M_rows` / `mask_rows` hold exactly the
// process' own rows [row0, row0 + nrows) of the tensor (its local_slabs
// consecutive slabs of the G-slab plan); halo rows arrive through the
// exchange, the global setup scalars through the upload's all-reduce.
void sharded_solve_rows(const Problem& p, const double* M_rows, const double* mask_rows,
                        const double* K_colmajor, const icnnm_solver_config* cfg,
                        int local_slabs, int world, int rank, const char* nccl_id128,
                        int device, double* L_out, int64_t* row0_out, int64_t* nrows_out,
                        icnnm_solve_report* report, std::chrono::steady_clock::time_point t0) {
  const int G = local_slabs * world;
  DeviceScope ds(device);
  Solver S;
  S.p = p;
  S.device = device;
  S.sharded = true;
  S.G = G;
  S.world = world;
  S.rank = rank;
  S.local = local_slabs;
  S.K.assign(K_colmajor, K_colmajor + static_cast<size_t>(p.k) * p.k);
  S.slabs.resize(local_slabs);
  for (int i = 0; i < local_slabs; ++i) {
    int64_t s = 0, c = 0;
    const int gi = rank * local_slabs + i;
    if (icnnm_shard_plan(p.dims[0], G, p.kd[0], gi, &s, &c) != ICNNM_OK) invalid(g_last_error);
    S.slabs[i].row0 = s;
    S.slabs[i].rows = c;
  }
  // world == 1 with an id: a one-rank communicator carries the exchange
  // (self send/recv + all-reduce), so the NCCL transport runs on one GPU
  if (world > 1 || nccl_id128) {
    if (!nccl_id128) invalid("sharded solve: NCCL unique id required for world > 1");
    S.comm = comm_create(nccl_id128, world, rank);
  }
  solver_alloc(S);
  solver_upload(S, M_rows, mask_rows);
  RunResult R = solver_run(S, *cfg);
  solver_download(S, L_out);
  if (row0_out) *row0_out = S.slabs[0].row0;
  if (nrows_out) {
    int64_t n = 0;
    for (auto& s : S.slabs) n += s.rows;
    *nrows_out = n;
  }
  double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  fill_report(S, *cfg, R, report, wall);
}

void rank_rows(const Problem& p, int local_slabs, int world, int rank, int64_t* row0,
               int64_t* nrows) {
  const int G = local_slabs * world;
  int64_t s0 = 0, c0 = 0, s1 = 0, c1 = 0;
  if (icnnm_shard_plan(p.dims[0], G, p.kd[0], rank * local_slabs, &s0, &c0) != ICNNM_OK ||
      icnnm_shard_plan(p.dims[0], G, p.kd[0], rank * local_slabs + local_slabs - 1, &s1, &c1) !=
          ICNNM_OK)
    invalid(g_last_error);
  *row0 = s0;
  *nrows = s1 + c1 - s0;
}
}  // namespace

int icnnm_sharded_rows(int order, const int64_t* dims, const int64_t* kdims, int local_slabs,
                       int world, int rank, int64_t* row0, int64_t* nrows) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    if (local_slabs < 1 || world < 1 || rank < 0 || rank >= world || !row0 || !nrows)
      invalid("sharded solve: bad slab / rank arguments");
    rank_rows(p, local_slabs, world, rank, row0, nrows);
  });
}

int icnnm_sharded_solve(int order, const int64_t* dims, const double* M_obs, const double* mask,
                        const int64_t* kdims, const double* K_colmajor,
                        const icnnm_solver_config* cfg, int local_slabs, int world, int rank,
                        const char* nccl_id128, int device, double* L_out, int64_t* row0_out,
                        int64_t* nrows_out, icnnm_solve_report* report) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    validate_cfg(cfg);
    Problem p = make_problem(order, dims, kdims);
    if (local_slabs < 1 || world < 1 || rank < 0 || rank >= world)
      invalid("sharded solve: bad slab / rank arguments");
    if (!L_out || !M_obs || !mask) invalid("null argument");
    validate_basis(p.k, K_colmajor, nullptr);
    int64_t r0 = 0, nr = 0;
    rank_rows(p, local_slabs, world, rank, &r0, &nr);
    const int64_t WT = p.dims[1] * p.dims[2];
    // the full tensor was passed: this rank reads (and validates) its own rows
    sharded_solve_rows(p, M_obs + r0 * WT, mask + r0 * WT, K_colmajor, cfg, local_slabs, world,
                       rank, nccl_id128, device, L_out, row0_out, nrows_out, report, t0);
  });
}

int icnnm_sharded_solve_local(int order, const int64_t* dims, int64_t row0, int64_t nrows,
                              const double* M_rows, const double* mask_rows,
                              const int64_t* kdims, const double* K_colmajor,
                              const icnnm_solver_config* cfg, int local_slabs, int world,
                              int rank, const char* nccl_id128, int device, double* L_out,
                              icnnm_solve_report* report) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    validate_cfg(cfg);
    Problem p = make_problem(order, dims, kdims);
    if (local_slabs < 1 || world < 1 || rank < 0 || rank >= world)
      invalid("sharded solve: bad slab / rank arguments");
    if (!L_out || !M_rows || !mask_rows) invalid("null argument");
    validate_basis(p.k, K_colmajor, nullptr);
    int64_t r0 = 0, nr = 0;
    rank_rows(p, local_slabs, world, rank, &r0, &nr);
    if (row0 != r0 || nrows != nr)
      invalid("sharded solve: rows [" + std::to_string(row0) + ", " + std::to_string(row0 + nrows) +
              ") are not this rank's slab rows [" + std::to_string(r0) + ", " +
              std::to_string(r0 + nr) + ") (icnnm_sharded_rows)");
    sharded_solve_rows(p, M_rows, mask_rows, K_colmajor, cfg, local_slabs, world, rank,
                       nccl_id128, device, L_out, nullptr, nullptr, report, t0);
  });
}

// --------------------------------------------------------------------------
// Probe
// --------------------------------------------------------------------------
int icnnm_probe_ffma_tflops(int device, double* out) {
  return guard([&] {
    if (!out) invalid("null argument");
    DeviceScope ds(device);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DBuf<float> o(1);
    const int iters = 1 << 16;
    const int blocks = sms * 8, threads = 256;
    icnnm_dev::icnnm_ffma_probe<<<blocks, threads>>>(o.p, 1024, 1.f);
    CKL();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    icnnm_dev::icnnm_ffma_probe<<<blocks, threads>>>(o.p, iters, 1.f);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 16.0 * iters * static_cast<double>(blocks) * threads;
    *out = flops / (ms * 1e-3) / 1e12;
  });
}


/* FP64 DFMA throughput in TFLOP/s (the Gram kernel's roofline denominator). */
int icnnm_probe_dfma_tflops(int device, double* out) {
  return guard([&] {
    if (!out) invalid("null argument");
    DeviceScope ds(device);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DBuf<double> o(1);
    const int iters = 1 << 14;
    const int blocks = sms * 8, threads = 256;
    icnnm_dev::icnnm_dfma_probe<<<blocks, threads>>>(o.p, 256, 1.0);
    CKL();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    icnnm_dev::icnnm_dfma_probe<<<blocks, threads>>>(o.p, iters, 1.0);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    *out = flops / (ms * 1e-3) / 1e12;
  });
}

}  // extern "C"
