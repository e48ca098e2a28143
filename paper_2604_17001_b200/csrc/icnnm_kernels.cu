// ICNNM per-iteration hot path: hand-written sm_100a kernels (FFMA engine).
//
// Kernel families (SURVEY.md §8a GPU mapping):
//   (a)+(b) icnnm_fwd_ffma   W <- A(L~)K + r c.W_old, fused column-norm^2
//   (c)     icnnm_adj_ffma   adj += A*( (W diag c) K^T )  (GEMM + col2im)
//   (d)     icnnm_update     P_Omega / L-update / multiplier bookkeeping
//           icnnm_coef       shrink factors c_j from the norms (prox_l21)
//   (e)     icnnm_gram_lags  autocorrelation lags for the Gram (fp64)
// The restated iteration (exact algebra of solver.cpp:107-126) is in
// DESIGN.md §2.
#include <cuda_runtime.h>
#include <cstdint>

#include "icnnm_kernels.cuh"

namespace icnnm_dev {

__device__ __forceinline__ int wrapi(int x, int n) {
  int r = x % n;
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Source/target buffer row for halo row `a` of a brick starting at h0.
__device__ __forceinline__ int halo_row(const Geo& g, int h0, int a) {
  int hs = h0 - (g.kh - 1) + a + g.hoff;
  return g.wrapH ? wrapi(hs, g.Hsrc) : hs;
}

__device__ __forceinline__ void brick_origin(const Geo& g, int blk, int& h0,
                                             int& w0, int& t0) {
  int bt_i = blk % g.nbt;
  int tmp = blk / g.nbt;
  int bw_i = tmp % g.nbw;
  int bh_i = tmp / g.nbw;
  h0 = bh_i * g.bh;
  w0 = bw_i * g.bw;
  t0 = bt_i * g.bt;
}

// Tap offsets inside the halo box: tapoff[s] = (sh*HW + sw)*HT + st, so that
// A[v, s] = halo[hidx(v) - tapoff[s]] with hidx(v) the halo index of voxel v
// shifted by (kh-1, kw-1, kt-1).  Padding taps point at offset 0.
__device__ __forceinline__ void fill_tapoff(const Geo& g, int* tapoff) {
  for (int s = threadIdx.x; s < g.ktp; s += blockDim.x) {
    int off = 0;
    if (s < g.k) {
      int st = s % g.kt;
      int q = s / g.kt;
      int sw = q % g.kw;
      int sh = q / g.kw;
      off = (sh * g.HW + sw) * g.HT + st;
    }
    tapoff[s] = off;
  }
}

// ---------------------------------------------------------------------------
// (a)+(b) forward implicit GEMM with fused epilogue.
//   mode 0: W = A(L~)K                  (initial / operator-level; no W read)
//   mode 1: W = A(L~)K + r c.W_old      (ADMM iteration; reads IterState)
// Columns are accumulated into norm2 (fp64) for the next prox.
// CTA = one brick (128 voxels) x all N-tiles; 128 threads, 8x8 micro-tiles
// (8 consecutive t-voxels x 8 columns).  The L~ halo brick is staged once in
// SMEM; K streams through a cp.async double buffer (L2-resident).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 4)
icnnm_fwd_ffma(Geo g, const float* __restrict__ Lt, const float* __restrict__ Krm,
               float* __restrict__ Wm, const float* __restrict__ cvec,
               const IterState* __restrict__ st, double* __restrict__ norm2,
               int mode) {
  float r = 0.f;
  if (mode == 1) {
    if (!st->active || st->it >= st->max_iters - 1) return;
    r = static_cast<float>(st->r);
  }
  if (mode == 2 && !st->active) return;  // exact residual: ||(1-c)W_t - A(L_{t+1})K||^2
  extern __shared__ float4 smem4[];
  float* Ks = reinterpret_cast<float*>(smem4);           // 2 * BK * BN
  int* tapoff = reinterpret_cast<int*>(Ks + 2 * BK * BN);  // ktp
  float* halo = reinterpret_cast<float*>(tapoff + g.ktp);  // HH*HW*HT
  __shared__ float red[4][BN];

  const int blk = blockIdx.x;
  int h0, w0, t0;
  brick_origin(g, blk, h0, w0, t0);
  const int tid = threadIdx.x;

  fill_tapoff(g, tapoff);
  {
    const int n = g.HH * g.HW * g.HT;
    for (int e = tid; e < n; e += blockDim.x) {
      int c = e % g.HT;
      int tmp = e / g.HT;
      int b = tmp % g.HW;
      int a = tmp / g.HW;
      int hs = halo_row(g, h0, a);
      hs = hs < 0 ? 0 : (hs >= g.Hsrc ? g.Hsrc - 1 : hs);
      int ws = wrapi(w0 - (g.kw - 1) + b, g.W);
      int ts = wrapi(t0 - (g.kt - 1) + c, g.T);
      halo[e] = __ldg(Lt + (static_cast<size_t>(hs) * g.W + ws) * g.T + ts);
    }
  }

  const int cg = tid & 7, vg = tid >> 3, lane = tid & 31, warp = tid >> 5;
  const int v0 = vg * 8;
  const int vt0 = v0 % g.bt;
  const int vw = (v0 / g.bt) % g.bw;
  const int vh = v0 / (g.bt * g.bw);
  const int hidx = ((vh + g.kh - 1) * g.HW + (vw + g.kw - 1)) * g.HT + (vt0 + g.kt - 1);
  const bool rowvalid = (h0 + vh < g.H) && (w0 + vw < g.W);
  const int ntiles = g.kp / BN;
  const int nchunks = g.ktp / BK;

  auto issue_k = [&](int buf, int ch, int nt) {
    float* dst = Ks + buf * BK * BN;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      int q = tid + 128 * p;
      int row = q >> 4, c4 = q & 15;
      cp_async16(dst + row * BN + c4 * 4,
                 Krm + static_cast<size_t>(ch * BK + row) * g.kp + nt * BN + c4 * 4);
    }
    cp_async_commit();
  };

  for (int nt = 0; nt < ntiles; ++nt) {
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    issue_k(0, 0, nt);
    for (int ch = 0; ch < nchunks; ++ch) {
      if (ch + 1 < nchunks) {
        issue_k((ch + 1) & 1, ch + 1, nt);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const float* kb = Ks + (ch & 1) * BK * BN + cg * 8;
      const int* to = tapoff + ch * BK;
#pragma unroll 4
      for (int s = 0; s < BK; ++s) {
        const float* ap = halo + (hidx - to[s]);
        float a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = ap[i];
        float4 b0 = *reinterpret_cast<const float4*>(kb + s * BN);
        float4 b1 = *reinterpret_cast<const float4*>(kb + s * BN + 4);
        float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }

    const int col0 = nt * BN + cg * 8;
    if (mode == 2) {
      float g2 = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool valid = rowvalid && (t0 + vt0 + i < g.T);
        const float* wp = Wm + (static_cast<size_t>(blk) * BM + v0 + i) * g.kp + col0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float gap = (1.f - cvec[col0 + j]) * wp[j] - acc[i][j];
          g2 = valid ? fmaf(gap, gap, g2) : g2;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g2 += __shfl_xor_sync(0xffffffffu, g2, o);
      if (lane == 0) atomicAdd(norm2, static_cast<double>(g2));
      continue;
    }
    // epilogue: W_new = acc + r c W_old, masked voxels -> 0, column norms.
    float cr[8];
    if (mode == 1) {
      float4 c0 = *reinterpret_cast<const float4*>(cvec + col0);
      float4 c1 = *reinterpret_cast<const float4*>(cvec + col0 + 4);
      cr[0] = r * c0.x; cr[1] = r * c0.y; cr[2] = r * c0.z; cr[3] = r * c0.w;
      cr[4] = r * c1.x; cr[5] = r * c1.y; cr[6] = r * c1.z; cr[7] = r * c1.w;
    }
    float nrm[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) nrm[j] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool valid = rowvalid && (t0 + vt0 + i < g.T);
      float* wp = Wm + (static_cast<size_t>(blk) * BM + v0 + i) * g.kp + col0;
      float w[8];
      if (mode == 1) {
        float4 o0 = *reinterpret_cast<const float4*>(wp);
        float4 o1 = *reinterpret_cast<const float4*>(wp + 4);
        float o[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = fmaf(cr[j], o[j], acc[i][j]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = acc[i][j];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        w[j] = valid ? w[j] : 0.f;
        nrm[j] = fmaf(w[j], w[j], nrm[j]);
      }
      *reinterpret_cast<float4*>(wp) = make_float4(w[0], w[1], w[2], w[3]);
      *reinterpret_cast<float4*>(wp + 4) = make_float4(w[4], w[5], w[6], w[7]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      nrm[j] += __shfl_xor_sync(0xffffffffu, nrm[j], 8);
      nrm[j] += __shfl_xor_sync(0xffffffffu, nrm[j], 16);
    }
    if (lane < 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) red[warp][lane * 8 + j] = nrm[j];
    }
    __syncthreads();
    if (tid < BN && norm2 != nullptr) {
      float s = red[0][tid] + red[1][tid] + red[2][tid] + red[3][tid];
      atomicAdd(norm2 + nt * BN + tid, static_cast<double>(s));
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// (c) adjoint: U = (W diag c) K^T on a brick x 64-tap tile (FFMA GEMM over
// j), scattered into an SMEM output brick (out[v - s] += U[v, s]); the brick
// (voxels shifted back by the kernel box) is flushed to adj with one fp32
// atomic per entry.  KT is [kp][ktp] (KT[j][s] = K[s][j]).
//   mode 0: c == nullptr -> 1 (operator-level conv_adjoint)
//   mode 1: ADMM iteration (reads IterState.active)
// ---------------------------------------------------------------------------
constexpr int WS_STRIDE = BM + 4;

__global__ void __launch_bounds__(128, 2)
icnnm_adj_ffma(Geo g, const float* __restrict__ Wm, const float* __restrict__ KT,
               const float* __restrict__ cvec, float* __restrict__ adj,
               const IterState* __restrict__ st, int mode) {
  if (mode == 1 && !st->active) return;
  extern __shared__ float4 smem4[];
  float* Ws = reinterpret_cast<float*>(smem4);          // BK * WS_STRIDE
  float* Ks = Ws + BK * WS_STRIDE;                       // 2 * BK * BN
  float* cs = Ks + 2 * BK * BN;                          // kp
  int* tapoff = reinterpret_cast<int*>(cs + g.kp);       // ktp
  float* obrick = reinterpret_cast<float*>(tapoff + g.ktp);  // HH*HW*HT

  const int blk = blockIdx.x;
  int h0, w0, t0;
  brick_origin(g, blk, h0, w0, t0);
  const int tid = threadIdx.x;
  const int nob = g.HH * g.HW * g.HT;
  for (int e = tid; e < nob; e += blockDim.x) obrick[e] = 0.f;
  for (int j = tid; j < g.kp; j += blockDim.x) cs[j] = cvec ? cvec[j] : (j < g.k ? 1.f : 0.f);
  fill_tapoff(g, tapoff);

  const int cg = tid & 7, vg = tid >> 3;
  const int v0 = vg * 8;
  const int vt0 = v0 % g.bt;
  const int vw = (v0 / g.bt) % g.bw;
  const int vh = v0 / (g.bt * g.bw);
  const int hidx = ((vh + g.kh - 1) * g.HW + (vw + g.kw - 1)) * g.HT + (vt0 + g.kt - 1);
  const int ntiles = g.ktp / BN;
  const int nchunks = g.kp / BK;
  const float* Wblk = Wm + static_cast<size_t>(blk) * BM * g.kp;

  auto load_w = [&](float4 (&wr)[8], int ch) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      int q = tid + 128 * p;
      int v = q >> 3, j4 = q & 7;
      wr[p] = __ldg(reinterpret_cast<const float4*>(Wblk + static_cast<size_t>(v) * g.kp +
                                                    ch * BK + j4 * 4));
    }
  };
  auto issue_k = [&](int buf, int ch, int nt) {
    float* dst = Ks + buf * BK * BN;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      int q = tid + 128 * p;
      int row = q >> 4, c4 = q & 15;
      cp_async16(dst + row * BN + c4 * 4,
                 KT + static_cast<size_t>(ch * BK + row) * g.ktp + nt * BN + c4 * 4);
    }
    cp_async_commit();
  };

  __syncthreads();
  for (int nt = 0; nt < ntiles; ++nt) {
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    float4 wr[8];
    load_w(wr, 0);
    issue_k(0, 0, nt);
    for (int ch = 0; ch < nchunks; ++ch) {
      __syncthreads();  // previous chunk's compute is done with Ws / Ks[(ch+1)&1]
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        int q = tid + 128 * p;
        int v = q >> 3, j4 = q & 7;
        int jb = ch * BK + j4 * 4;
        float* d = Ws + (j4 * 4) * WS_STRIDE + v;
        d[0] = wr[p].x * cs[jb];
        d[WS_STRIDE] = wr[p].y * cs[jb + 1];
        d[2 * WS_STRIDE] = wr[p].z * cs[jb + 2];
        d[3 * WS_STRIDE] = wr[p].w * cs[jb + 3];
      }
      if (ch + 1 < nchunks) {
        issue_k((ch + 1) & 1, ch + 1, nt);
        load_w(wr, ch + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const float* kb = Ks + (ch & 1) * BK * BN + cg * 8;
      const float* wb = Ws + vg * 8;
#pragma unroll 4
      for (int j = 0; j < BK; ++j) {
        float4 a0 = *reinterpret_cast<const float4*>(wb + j * WS_STRIDE);
        float4 a1 = *reinterpret_cast<const float4*>(wb + j * WS_STRIDE + 4);
        float4 b0 = *reinterpret_cast<const float4*>(kb + j * BN);
        float4 b1 = *reinterpret_cast<const float4*>(kb + j * BN + 4);
        float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) acc[i][jj] = fmaf(a[i], b[jj], acc[i][jj]);
      }
    }
    // col2im scatter into the SMEM output brick.
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      int s = nt * BN + cg * 8 + jj;
      if (s < g.k) {
        int base = hidx - tapoff[s];
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicAdd(obrick + base + i, acc[i][jj]);
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < nob; e += blockDim.x) {
    float v = obrick[e];
    if (v == 0.f) continue;
    int c = e % g.HT;
    int tmp = e / g.HT;
    int b = tmp % g.HW;
    int a = tmp / g.HW;
    int hs = halo_row(g, h0, a);
    if (hs < 0 || hs >= g.Hsrc) continue;
    int ws = wrapi(w0 - (g.kw - 1) + b, g.W);
    int ts = wrapi(t0 - (g.kt - 1) + c, g.T);
    atomicAdd(adj + (static_cast<size_t>(hs) * g.W + ws) * g.T + ts, v);
  }
}

// ---------------------------------------------------------------------------
// Block reduction helper (fp64).
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void block_reduce_add(double (&v)[N], double* dst) {
  __shared__ double sh[32][N];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < N; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < N; ++q) sh[warp][q] = v[q];
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double x = lane < nw ? sh[lane][q] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0 && dst != nullptr) atomicAdd(dst + q, x);
    }
  }
}

// ---------------------------------------------------------------------------
// Deterministic reductions.  The forward kernel writes one row of column
// partials per CTA, the update kernel one row of its 5 report sums per block,
// the exact-residual forward one gap partial per CTA; these fold them in a
// fixed order (thread t sums rows t, t + blockDim, ... sequentially, then a
// fixed shuffle tree and a fixed sum over warps), so a solve is bit-for-bit
// reproducible run to run (the reference is deterministic).
// ---------------------------------------------------------------------------
__device__ double block_sum_fixed(double v) {
  __shared__ double sh[32];
  __shared__ double out;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // sh / out reuse across calls
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sh[w];
    out = t;
  }
  __syncthreads();
  return out;
}

// Fixed-order sums of up to NV values per thread over the block: shuffle tree
// within each warp, then thread 0 adds the warps in order.
template <int NV>
__device__ void block_sum_fixed_n(double (&v)[NV], double* out) {
  __shared__ double sh[NV][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  __syncthreads();  // sh reuse across calls
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) sh[q][warp] = v[q];
  __syncthreads();
  if (threadIdx.x < NV) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sh[threadIdx.x][w];
    out[threadIdx.x] = t;
  }
}

__device__ void fold_partials(const Partials& P, int kp, double* red) {
  if (P.npart != nullptr) {
    // column j: FOLD_Q threads, thread q sums rows r = q, q + FOLD_Q, ... in
    // order (loads issued in batches of 8 ahead of the adds), then the FOLD_Q
    // partials are added in order -- a fixed summation tree whatever the launch
    constexpr int FOLD_Q = 4;
    __shared__ double fq[FOLD_Q][256];
    for (int j0 = 0; j0 < kp; j0 += 256) {
      const int jl = threadIdx.x & 255, q = threadIdx.x >> 8;  // blockDim.x = 1024
      const int j = j0 + jl;
      double t = 0.0;
      if (j < kp && q < FOLD_Q) {
        const double* src = P.npart + j;
        int r = q;
        for (; r + 7 * FOLD_Q < P.nrows; r += 8 * FOLD_Q) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = src[static_cast<size_t>(r + u * FOLD_Q) * kp];
#pragma unroll
          for (int u = 0; u < 8; ++u) t += v[u];
        }
        for (; r < P.nrows; r += FOLD_Q) t += src[static_cast<size_t>(r) * kp];
      }
      __syncthreads();
      if (q < FOLD_Q) fq[q][jl] = t;
      __syncthreads();
      if (q == 0 && j < kp) red[j] = (fq[0][jl] + fq[1][jl]) + (fq[2][jl] + fq[3][jl]);
    }
  }
  double* slot = red + kp;
  if (P.upart != nullptr) {
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int r = threadIdx.x; r < P.urows; r += blockDim.x) {
      const double* u = P.upart + static_cast<size_t>(r) * 8;
#pragma unroll
      for (int q = 0; q < 5; ++q) v[q] += u[q];
    }
    block_sum_fixed_n<5>(v, slot);
  }
  if (P.gpart != nullptr) {
    double v[1] = {0.0};
    for (int r = threadIdx.x; r < P.grows; r += blockDim.x) v[0] += P.gpart[r];
    block_sum_fixed_n<1>(v, slot + 5);
  }
  __syncthreads();
}

// Sharded solves fold before the cross-rank all-reduce of `red`.
__global__ void icnnm_fold(Partials P, int kp, double* red) {
  pdl_wait();
  pdl_trigger();
  fold_partials(P, kp, red);
}

// Deterministic adjoint output: the tcgen05 adjoint adds each brick's partial
// sums into adjq as {hi, lo} fp32 pairs on fixed grids (adj_grid,
// icnnm_kernels.cuh: every add is exact, so the result does not depend on the
// order in which CTAs flush).  This folds the pairs into fp32 adj and clears
// the accumulator for the next launch.
__global__ void __launch_bounds__(256)
icnnm_adj_q2f(int64_t n, const IterState* __restrict__ st, float2* __restrict__ adjq,
              float* __restrict__ adj) {
  pdl_wait();
  pdl_trigger();
  if (!st->active) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float2 q = adjq[i];
  adjq[i] = make_float2(0.f, 0.f);
  adj[i] = static_cast<float>(static_cast<double>(q.x) + static_cast<double>(q.y));
}

// ---------------------------------------------------------------------------
// Shrink coefficients (prox_l21, solver.cpp:42-50, folded): c_j = tau/n_j if
// n_j > tau else 1, tau = 1/theta.  Also evaluates the stopping test of the
// previous iteration (solver.cpp:136-139) and advances the iteration state.
// Single CTA.
// ---------------------------------------------------------------------------
__global__ void icnnm_coef(IterState* st, const double* __restrict__ theta,
                           double* __restrict__ red, float* __restrict__ cvec,
                           IterStats* __restrict__ stats, int k, int kp, double kd,
                           double res_scale, double tol_p, double tol_c, double floor_rel,
                           int exact, Partials P) {
  pdl_wait();
  pdl_trigger();
  // deterministic mode: fold the per-CTA / per-block partials of the
  // iteration that just finished into red (fixed order)
  fold_partials(P, kp, red);
  // red = [norm2 (kp) | update slot (dl2, l2o, fit, ip, ln2) | pad]
  __shared__ int go;
  __shared__ int cur;
  if (threadIdx.x == 0) {
    int it = st->next_it;
    int g = st->active;
    if (g && it > 0) {
      IterStats& p = stats[it - 1];
      double* slot = red + kp;
      p.dl2 = slot[0]; p.l2o = slot[1]; p.fit = slot[2]; p.ip = slot[3]; p.ln2 = slot[4];
      p.gap2 = slot[5];
      for (int q = 0; q < 8; ++q) slot[q] = 0.0;
      double gap2 = exact ? p.gap2 : p.z2 - 2.0 * p.ip + kd * p.ln2;
      double scale2 = p.z2 + kd * p.ln2;
      double res = sqrt(fmax(gap2, 0.0)) / res_scale;
      // identity form: below the floor the gap is unresolved in fp32
      bool res_ok = exact ? true : gap2 > floor_rel * scale2;
      double lc = sqrt(p.dl2) / fmax(sqrt(p.l2o), 1e-300);
      if ((res_ok && res < tol_p) || lc < tol_c) {
        g = 0;
        st->converged = 1;
      }
    }
    if (g && it >= st->max_iters) g = 0;
    if (g) {
      st->it = it;
      st->next_it = it + 1;
      st->theta = theta[it];
      st->r = theta[it] / theta[it + 1];
    }
    st->active = g;
    go = g;
    cur = it;
  }
  __syncthreads();
  if (!go) return;
  const double th = theta[cur];
  const double tau = 1.0 / th;
  double acc[2] = {0.0, 0.0};
  double amax = 0.0;  // max_j c_j n_j = max_j min(n_j, tau) bounds |W_vj c_j|
  for (int j = threadIdx.x; j < kp; j += blockDim.x) {
    double n = sqrt(red[j]);
    red[j] = 0.0;
    float c = 0.f;
    if (j < k) {
      double cd = (n > tau) ? tau / n : 1.0;
      c = static_cast<float>(cd);
      acc[0] += fmax(0.0, n - tau);
      acc[1] += (1.0 - cd) * (1.0 - cd) * n * n;
      amax = fmax(amax, fmin(n, tau));
    }
    cvec[j] = c;
  }
  {
    __shared__ double wmax[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = amax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, wmax[w]);
      st->adj_amax = m;
    }
  }
  block_reduce_add<2>(acc, &stats[cur].l21);
}

// ---------------------------------------------------------------------------
// (d) fused elementwise update (solver.cpp:112-126 restated):
//   D  = (lambda (pm - mask L) - (theta/k) adj) / (lambda mask + theta)
//   L <- L + D ;  L~ = L + r D (forward input) ;  adj <- 0
//   V <- r (k L_old - adj - k L_new)           (V = A*(Y/theta K^T))
// plus the fp64 partial sums of the report (fit, ||D||, ||L||, residual).
// ---------------------------------------------------------------------------
// One resident wave (grid = SMs x resident blocks, host); each thread loads
// UPD_U elements (stride = grid size) before computing, so every thread keeps
// 5 x UPD_U independent loads in flight (the one-element-per-thread form was
// latency-bound at 34 us for 27 MB at config 2: long-scoreboard stalls, 5% of
// HBM bandwidth).
__global__ void __launch_bounds__(256)
icnnm_update(int64_t m, const IterState* __restrict__ st, double lambda, double kd,
             float* __restrict__ adj, double* __restrict__ L, double* __restrict__ V,
             const float* __restrict__ pm, const float* __restrict__ mask,
             float* __restrict__ Lt, double* __restrict__ slot, float* __restrict__ Lr,
             double* __restrict__ upart, float2* __restrict__ adjq) {
  pdl_wait();
  pdl_trigger();
  if (!st->active) return;
  const double th = st->theta;
  const double r = st->r;
  const double ck = th / kd;
  double acc[5] = {0, 0, 0, 0, 0};  // dl2, l2o, fit, ip, ln2
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < m;
       i0 += UPD_U * stride) {
    float a_[UPD_U], mk_[UPD_U], p_[UPD_U];
    double lo_[UPD_U], v_[UPD_U];
#pragma unroll
    for (int u = 0; u < UPD_U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < m) {
        if (adjq != nullptr) {
          // deterministic adjoint, unsharded: fold the {hi, lo} grid pair here
          // (the rounding of icnnm_adj_q2f) and clear it for the next launch
          const float2 q = adjq[i];
          a_[u] = static_cast<float>(static_cast<double>(q.x) + static_cast<double>(q.y));
        } else {
          a_[u] = adj[i];
        }
        lo_[u] = L[i];
        mk_[u] = mask[i];
        p_[u] = pm[i];
        v_[u] = V[i];
      }
    }
#pragma unroll
    for (int u = 0; u < UPD_U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= m) break;
      const double a = a_[u];
      const double lo = lo_[u];
      const double mk = mk_[u];
      const double p = p_[u];
      const double d = (lambda * (p - mk * lo) - ck * a) / (lambda * mk + th);
      const double ln = lo + d;
      const double v = v_[u];
      L[i] = ln;
      Lt[i] = static_cast<float>(ln + r * d);
      if (Lr != nullptr) Lr[i] = static_cast<float>(ln);
      if (adjq != nullptr)
        adjq[i] = make_float2(0.f, 0.f);
      else
        adj[i] = 0.f;
      V[i] = r * (kd * lo - a - kd * ln);
      const double f = mk * (ln - p);
      acc[0] += d * d;
      acc[1] += lo * lo;
      acc[2] += f * f;
      acc[3] += (kd * lo - v - a) * ln;
      acc[4] += ln * ln;
    }
  }
  if (upart != nullptr) {
    // deterministic: this block's sums in its own row (fixed-order tree)
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double v = block_sum_fixed(acc[q]);
      if (threadIdx.x == 0) upart[blockIdx.x * 8 + q] = v;
    }
    return;
  }
  block_reduce_add<5>(acc, slot);
}

// Setup: pm = M.mask (f32), mask (f32), L0 (f64, zero or mean fill), L~ = L0,
// V = 0; also |pm| max and ||pm||^2 for theta0 / res_scale.
__global__ void icnnm_setup(int64_t m, const double* __restrict__ M, const double* __restrict__ msk,
                            int mean_fill, double mean, float* __restrict__ pm,
                            float* __restrict__ maskf, double* __restrict__ L,
                            double* __restrict__ V, float* __restrict__ Lt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double mk = msk[i];
    const double p = M[i] * mk;
    double l = p;
    if (mean_fill) l += (1.0 - mk) * mean;
    pm[i] = static_cast<float>(p);
    maskf[i] = static_cast<float>(mk);
    L[i] = l;
    V[i] = 0.0;
    Lt[i] = static_cast<float>(l);
  }
}

// ---------------------------------------------------------------------------
// (e) Gram lags (fp64): R[d] = sum_i X[i] X[(i - d) mod dims] for
// d in [-(kh-1), kh-1] x [-(kw-1), kw-1] x [-(kt-1), kt-1]
// (= circular_autocorrelation, fft.cpp:109-118, at the lags conv_gram reads,
// spectral.cpp:69-79).  grid.x = 2kh-1 (dh), grid.y strides over bricks.
// Each CTA stages rows h-dh of its brick with a +-(kw-1, kt-1) halo.
// ---------------------------------------------------------------------------
constexpr int GRAM_LPT = 8;
__global__ void __launch_bounds__(256)
icnnm_gram_lags(int H, int W, int T, int kh, int kw, int kt, int bh, int bw, int bt,
                const double* __restrict__ X, double* __restrict__ R) {
  extern __shared__ double gsm[];
  const int dh = static_cast<int>(blockIdx.x) - (kh - 1);
  const int HWd = bw + 2 * (kw - 1), HTd = bt + 2 * (kt - 1);
  const int nbh = (H + bh - 1) / bh, nbw = (W + bw - 1) / bw, nbt = (T + bt - 1) / bt;
  const int nb = nbh * nbw * nbt;
  double* own = gsm;                       // bh*bw*bt
  double* hal = gsm + bh * bw * bt;        // bh*HWd*HTd
  const int nlw = 2 * kw - 1, nlt = 2 * kt - 1, nl = nlw * nlt;
  double acc[GRAM_LPT];
#pragma unroll
  for (int p = 0; p < GRAM_LPT; ++p) acc[p] = 0.0;
  for (int b = blockIdx.y; b < nb; b += gridDim.y) {
    const int bt_i = b % nbt, bw_i = (b / nbt) % nbw, bh_i = b / (nbt * nbw);
    const int h0 = bh_i * bh, w0 = bw_i * bw, t0 = bt_i * bt;
    __syncthreads();
    for (int e = threadIdx.x; e < bh * bw * bt; e += blockDim.x) {
      int c = e % bt, bb = (e / bt) % bw, a = e / (bt * bw);
      int h = h0 + a, w = w0 + bb, t = t0 + c;
      own[e] = (h < H && w < W && t < T) ? X[(static_cast<size_t>(h) * W + w) * T + t] : 0.0;
    }
    for (int e = threadIdx.x; e < bh * HWd * HTd; e += blockDim.x) {
      int c = e % HTd, bb = (e / HTd) % HWd, a = e / (HTd * HWd);
      int h = wrapi(h0 + a - dh, H);
      int w = wrapi(w0 + bb - (kw - 1), W);
      int t = wrapi(t0 + c - (kt - 1), T);
      hal[e] = X[(static_cast<size_t>(h) * W + w) * T + t];
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < GRAM_LPT; ++p) {
      const int l = threadIdx.x + p * blockDim.x;
      if (l < nl) {
        const int dw = l / nlt - (kw - 1), dt = l % nlt - (kt - 1);
        double s = 0.0;
        for (int a = 0; a < bh; ++a)
          for (int bb = 0; bb < bw; ++bb) {
            const double* o = own + (a * bw + bb) * bt;
            const double* hp = hal + (a * HWd + bb - dw + (kw - 1)) * HTd - dt + (kt - 1);
            for (int c = 0; c < bt; ++c) s = fma(o[c], hp[c], s);
          }
        acc[p] += s;
      }
    }
  }
  // deterministic: one partial per (dh, CTA-row); icnnm_gram_reduce sums them
  // in a fixed order, so learn_basis is bit-reproducible run to run
#pragma unroll
  for (int p = 0; p < GRAM_LPT; ++p) {
    const int l = threadIdx.x + p * blockDim.x;
    if (l < nl)
      R[(static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * nl + l] = acc[p];
  }
}

// ---------------------------------------------------------------------------
// (e) Gram lags, register-tiled (fp64), for kt <= GRAM_KT_MAX.
// Only the lags with dh >= 0 are computed (grid.x = kh): R[-d] = R[d] for the
// circular autocorrelation of a real tensor, mirrored by icnnm_gram_reduce_sym.
// Brick = bh x bw x bt voxels (RS = bh bw "rows" of bt frames) with a halo of
// +-(kw-1) columns and +-(kt-1) frames, rows shifted by -dh.  Thread (dw, rs)
// computes all NLT = 2kt-1 frame lags of the 1-D correlation of own row rs
// with halo row rs - dw: per 4 frames 4 own loads + 4 halo loads feed 4 NLT
// DFMAs from a sliding register window (the lag-per-thread kernel above needs
// two shared-memory loads per DFMA).  Per-thread sums are reduced over rs in a
// fixed order at the end (deterministic, like the partial rows).
// ---------------------------------------------------------------------------
template <int KT>
__global__ void __launch_bounds__(256, (KT <= 6 ? 2 : 1))
icnnm_gram_lags_rt(int H, int W, int T, int kw, int bh, int bw, int bt,
                   const double* __restrict__ X, double* __restrict__ R) {
  constexpr int NLT = 2 * KT - 1;
  // frames per step: the window of CW + NLT - 1 halo frames lives in two
  // register arrays of CW that swap roles every step (no register shifting)
  constexpr int CW = (NLT - 1) < 2 ? 2 : (NLT - 1);
  extern __shared__ double gsm[];
  const int dh = static_cast<int>(blockIdx.x);
  const int nlw = 2 * kw - 1;
  const int RS = bh * bw;
  const int HWd = bw + 2 * (kw - 1);
  const int btp = (bt + 2 * CW - 1) / (2 * CW) * (2 * CW);
  const int po = btp + 2;                 // own row pitch (rows of one warp: <= 3 distinct)
  const int hl = btp + CW;                // halo row length (>= btp + 2 (KT - 1))
  const int ph = hl | 1;                  // odd pitch: a half-warp's rows hit distinct banks
  double* own = gsm;                      // RS * po
  double* hal = gsm + RS * po;            // bh * HWd * ph
  const int nbh = (H + bh - 1) / bh, nbw = (W + bw - 1) / bw, nbt = (T + bt - 1) / bt;
  const int nb = nbh * nbw * nbt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int dwi = static_cast<int>(threadIdx.x) % nlw, rs = static_cast<int>(threadIdx.x) / nlw;
  const bool act = rs < RS;
  const int ra = act ? rs / bw : 0, rb = act ? rs % bw : 0;
  const double* orow = own + (act ? rs : 0) * po;
  const double* hrow = hal + (ra * HWd + rb - dwi + 2 * (kw - 1)) * ph;
  double acc[NLT];
#pragma unroll
  for (int d = 0; d < NLT; ++d) acc[d] = 0.0;
  // one step: own frames c0 .. c0+CW-1 against the window lo ++ hi
  // (lo = halo frames c0 .. c0+CW-1, hi = the next CW); lag index
  // d = dt + (kt-1): own[c] pairs with halo frame c + NLT-1-d
  auto step = [&](const double (&o)[CW], const double (&lo)[CW], const double (&hi)[CW]) {
#pragma unroll
    for (int i = 0; i < CW; ++i)
#pragma unroll
      for (int d = 0; d < NLT; ++d) {
        const int u = i + NLT - 1 - d;
        acc[d] = fma(o[i], u < CW ? lo[u] : hi[u - CW], acc[d]);
      }
  };
  // brick b's own rows and halo into buffer `buf` with 8-byte cp.async copies
  // (a warp per row: the row's (h, w) once, frames across the lanes); the next
  // brick's copies fly while the current one is computed
  const int tile = RS * po + bh * HWd * ph;
  auto load = [&](int b, int buf) {
    const int bt_i = b % nbt, bw_i = (b / nbt) % nbw, bh_i = b / (nbt * nbw);
    const int h0 = bh_i * bh, w0 = bw_i * bw, t0 = bt_i * bt;
    double* ownb = own + buf * tile;
    double* halb = hal + buf * tile;
    for (int r = warp; r < RS; r += 8) {
      const int h = h0 + r / bw, w = w0 + r % bw;
      const bool in = h < H && w < W;
      const double* src = X + (static_cast<size_t>(in ? h : 0) * W + (in ? w : 0)) * T + t0;
      for (int c = lane; c < btp; c += 32) {
        if (in && c < bt && t0 + c < T)
          cp_async8(ownb + r * po + c, src + c);
        else
          ownb[r * po + c] = 0.0;
      }
    }
    for (int q = warp; q < bh * HWd; q += 8) {
      const int h = wrapi(h0 + q / HWd - dh, H);
      const int w = wrapi(w0 + q % HWd - (kw - 1), W);
      const double* src = X + (static_cast<size_t>(h) * W + w) * T;
      for (int c = lane; c < hl; c += 32) {
        int t = t0 + c - (KT - 1);
        t = t < 0 ? t + T : t;
        t = t >= T ? t - T : t;
        if (static_cast<unsigned>(t) >= static_cast<unsigned>(T)) t = wrapi(t, T);
        cp_async8(halb + q * ph + c, src + t);
      }
    }
    cp_async_commit();
  };
  int buf = 0;
  if (static_cast<int>(blockIdx.y) < nb) load(blockIdx.y, 0);
  for (int b = blockIdx.y; b < nb; b += gridDim.y, buf ^= 1) {
    const int bn = b + static_cast<int>(gridDim.y);
    if (bn < nb) {
      load(bn, buf ^ 1);   // its previous reader finished before the barrier below
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (act) {
      const double* orw = orow + buf * tile;
      const double* hrw = hrow + buf * tile;
      double wa[CW], wb[CW], o[CW];
#pragma unroll
      for (int u = 0; u < CW; ++u) wa[u] = hrw[u];
      for (int c0 = 0; c0 < btp; c0 += 2 * CW) {
#pragma unroll
        for (int u = 0; u < CW; ++u) {
          wb[u] = hrw[c0 + CW + u];
          o[u] = orw[c0 + u];
        }
        step(o, wa, wb);
#pragma unroll
        for (int u = 0; u < CW; ++u) {
          wa[u] = hrw[c0 + 2 * CW + u];   // last step: zero-padded frames of the pitch
          o[u] = orw[c0 + CW + u];
        }
        step(o, wb, wa);
      }
    }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's load
  }
  // fixed-order reduction over rs: red[rs][dw][d] in shared memory
  __syncthreads();
  double* red = gsm;
  if (act)
#pragma unroll
    for (int d = 0; d < NLT; ++d) red[(rs * nlw + dwi) * NLT + d] = acc[d];
  __syncthreads();
  const int nl = nlw * NLT;
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < RS; ++r) s += red[r * nl + l];
    R[(static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * nl + l] = s;
  }
}

// The instantiation for frame-kernel size kt, or null (kt > GRAM_KT_MAX).
void* gram_lags_rt_ptr(int kt) {
  switch (kt) {
    case 1: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<1>);
    case 2: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<2>);
    case 3: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<3>);
    case 4: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<4>);
    case 5: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<5>);
    case 6: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<6>);
    case 7: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<7>);
    case 8: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<8>);
    case 9: return reinterpret_cast<void*>(&icnnm_gram_lags_rt<9>);
    default: return nullptr;
  }
}

// Half-space partials [ny][kh][nl] (dh = 0..kh-1) -> the full lag box
// R_out[(2kh-1)][nl] += sum_y (fixed order), mirrored: R[-dh][-dw][-dt] =
// R[dh][dw][dt] (index nl-1-l in row kh-1-dh); in the dh = 0 row the upper
// half (l >= centre) is mirrored onto the lower, so R is exactly symmetric.
__global__ void icnnm_gram_reduce_sym(int kh, int nl, int ny, const double* __restrict__ partial,
                                      double* __restrict__ R_out) {
  const int64_t n = static_cast<int64_t>(kh) * nl;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int y = 0; y < ny; ++y) s += partial[static_cast<size_t>(y) * n + i];
    const int dh = static_cast<int>(i / nl), l = static_cast<int>(i % nl);
    if (dh == 0) {
      if (l < (nl - 1) / 2) continue;
      R_out[static_cast<size_t>(kh - 1) * nl + l] += s;
      if (l != (nl - 1) / 2) R_out[static_cast<size_t>(kh - 1) * nl + (nl - 1 - l)] += s;
    } else {
      R_out[static_cast<size_t>(kh - 1 + dh) * nl + l] += s;
      R_out[static_cast<size_t>(kh - 1 - dh) * nl + (nl - 1 - l)] += s;
    }
  }
}

// FP64 DFMA peak probe: independent FMA chains in registers.
__global__ void __launch_bounds__(256) icnnm_dfma_probe(double* out, int iters, double seed) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-9 + i;
  const double b = 0.999999, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

// R_out[i] += sum_y partial[y][i] (fixed order)
__global__ void icnnm_gram_reduce(int64_t n, int ny, const double* __restrict__ partial,
                                  double* __restrict__ R_out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int y = 0; y < ny; ++y) s += partial[static_cast<size_t>(y) * n + i];
    R_out[i] += s;
  }
}

// ---------------------------------------------------------------------------
// Operator-level helpers.
// ---------------------------------------------------------------------------
__global__ void icnnm_colnorm2(int64_t rows, int64_t cols, const double* __restrict__ W,
                               double* __restrict__ out) {
  // one CTA per column, column-major W
  const int64_t c = blockIdx.x;
  double acc[1] = {0.0};
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    double v = W[c * rows + i];
    acc[0] += v * v;
  }
  block_reduce_add<1>(acc, out + c);
}

__global__ void icnnm_colscale(int64_t rows, int64_t cols, const double* __restrict__ W,
                               const double* __restrict__ n2, double tau,
                               double* __restrict__ Z) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * cols;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = i / rows;
    const double n = sqrt(n2[c]);
    Z[i] = W[i] * ((n > tau) ? (1.0 - tau / n) : 0.0);
  }
}

__global__ void icnnm_f64_to_f32(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    b[i] = static_cast<float>(a[i]);
}

// Reverse halo accumulate: dst[i] += src[i]; src[i] = 0 (adjoint partial
// sums of rows owned by the previous slab).
__global__ void icnnm_add_rows(int64_t n, float* __restrict__ dst, float* __restrict__ src) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    dst[i] += src[i];
    src[i] = 0.f;
  }
}

// FP32 FFMA peak probe: independent FMA chains in registers.
__global__ void __launch_bounds__(256) icnnm_ffma_probe(float* out, int iters, float seed) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed + threadIdx.x * 1e-7f + i;
  const float b = 0.999999f, c = 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678f) out[0] = s;
}

}  // namespace icnnm_dev
