// Recovery-theory diagnostics on the GPU: the `analyze`
// path of the reference (/root/reference/proj/core/src/analysis.cpp),
// matrix-free.
//
// The reference forms the dense m x k convolution matrix A(L0) and runs an
// Eigen BDCSVD on it (analysis.cpp:111-135), and evaluates k FFT convolutions
// for the relative eigenvalues (:29-38).  Here every quantity comes from
// fp64 implicit GEMMs over the halo brick (the m x k matrix is never
// materialised) plus k x k host/GPU algebra:
//
//   sigma^K_i   = ||A(L0) K_i||                     icnnm_conv64, column norms
//   alpha_K^2   = top eig of (K_I D)^T G (K_I D)    conv Gram (icnnm_gram_lags),
//                                                   icnnm_dgemm_tn, host power
//                                                   iteration (:51-69, :79-96)
//   conv_coherence: streaming TSQR of A(L0) (row blocks gathered on the GPU
//                 by icnnm_im2col64, cuSOLVER geqrf), SVD of the k x k R
//                 (cuSOLVER gesvd) -> s, V, both backward stable like the
//                 reference's BDCSVD (a Gram eigensolve would square the
//                 condition number and lose the singular vectors near the
//                 1e-8 rank cut); mu2 from the rows of V_r;
//                 mu1 = m/r max_v ||(A V_r S_r^-1)_v||^2 (icnnm_conv64,
//                 row-norm epilogue) (:111-135)
//   thresholds, active coherence: closed forms on the host (:98-109, :137-153)
//
// Everything is fp64: these are one-time diagnostics whose rank decisions use
// a 1e-8 relative tolerance (spectral.hpp:25), below fp32 resolution.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "icnnm_host_common.h"

namespace icnnm_dev {

constexpr int C64_BN = 64;  // basis columns per N-tile
constexpr int C64_BK = 32;  // taps per staged chunk

__device__ __forceinline__ int wrap64(int x, int n) {
  int r = x % n;
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ void cp_async16_64(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// out[v, c] = sum_s L[(v - s) mod dims] B[s, c]   (fp64, one CTA per brick)
//   mode 0: part[blk * np + c] = sum over the brick's voxels of out[v, c]^2
//   mode 1: part[blk]          = max over the brick's voxels of sum_c out[v, c]^2
// B is tap-major [ktp][np], zero padded.  256 threads: lane&15 picks 4
// columns of the 64-wide N-tile, (warp, lane>>4) picks 8 consecutive-t voxels.
__global__ void __launch_bounds__(256)
icnnm_conv64(Geo g, int np, const double* __restrict__ L, const double* __restrict__ Bp,
             double* __restrict__ part, int mode) {
  extern __shared__ double2 smem2[];
  double* Ks = reinterpret_cast<double*>(smem2);                    // 2 * BK * BN
  int* tapoff = reinterpret_cast<int*>(Ks + 2 * C64_BK * C64_BN);  // ktp
  double* halo = reinterpret_cast<double*>(tapoff + ((g.ktp + 1) & ~1));
  __shared__ double red[8][C64_BN];

  const int blk = blockIdx.x;
  const int bt_i = blk % g.nbt, tmp = blk / g.nbt;
  const int h0 = (tmp / g.nbw) * g.bh, w0 = (tmp % g.nbw) * g.bw, t0 = bt_i * g.bt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int s = tid; s < g.ktp; s += blockDim.x) {
    int off = 0;
    if (s < g.k) {
      const int st = s % g.kt, q = s / g.kt;
      off = ((q / g.kw) * g.HW + (q % g.kw)) * g.HT + st;
    }
    tapoff[s] = off;
  }
  {
    const int n = g.HH * g.HW * g.HT;
    for (int e = tid; e < n; e += blockDim.x) {
      const int c = e % g.HT, r2 = e / g.HT;
      const int b = r2 % g.HW, a = r2 / g.HW;
      const int hs = wrap64(h0 - (g.kh - 1) + a, g.H);
      const int ws = wrap64(w0 - (g.kw - 1) + b, g.W);
      const int ts = wrap64(t0 - (g.kt - 1) + c, g.T);
      halo[e] = L[(static_cast<size_t>(hs) * g.W + ws) * g.T + ts];
    }
  }

  const int cg = lane & 15;
  const int vg = warp * 2 + (lane >> 4);
  const int v0 = vg * 8;
  const int vt0 = v0 % g.bt;
  const int vw = (v0 / g.bt) % g.bw;
  const int vh = v0 / (g.bt * g.bw);
  const int hidx = ((vh + g.kh - 1) * g.HW + (vw + g.kw - 1)) * g.HT + (vt0 + g.kt - 1);
  const bool rowvalid = (h0 + vh < g.H) && (w0 + vw < g.W);
  bool valid[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) valid[i] = rowvalid && (t0 + vt0 + i < g.T);

  const int ntiles = np / C64_BN;
  const int nchunks = g.ktp / C64_BK;
  auto issue = [&](int buf, int ch, int nt) {
    double* dst = Ks + buf * C64_BK * C64_BN;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int q = tid + 256 * p;  // 1024 16-byte pieces
      const int row = q >> 5, c2 = q & 31;
      cp_async16_64(dst + row * C64_BN + c2 * 2,
                    Bp + static_cast<size_t>(ch * C64_BK + row) * np + nt * C64_BN + c2 * 2);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  double rowacc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) rowacc[i] = 0.0;

  for (int nt = 0; nt < ntiles; ++nt) {
    double acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    __syncthreads();  // halo/tapoff ready; previous tile's Ks reads done
    issue(0, 0, nt);
    for (int ch = 0; ch < nchunks; ++ch) {
      if (ch + 1 < nchunks) {
        issue((ch + 1) & 1, ch + 1, nt);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      __syncthreads();
      const double* kb = Ks + (ch & 1) * C64_BK * C64_BN + cg * 4;
      const int* to = tapoff + ch * C64_BK;
#pragma unroll 4
      for (int s = 0; s < C64_BK; ++s) {
        const double* ap = halo + (hidx - to[s]);
        double a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = ap[i];
        const double2 b01 = *reinterpret_cast<const double2*>(kb + s * C64_BN);
        const double2 b23 = *reinterpret_cast<const double2*>(kb + s * C64_BN + 2);
        const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }

    if (mode == 0) {
      double cs[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += valid[i] ? acc[i][j] * acc[i][j] : 0.0;
        s += __shfl_xor_sync(0xffffffffu, s, 16);
        cs[j] = s;
      }
      if (lane < 16) {
#pragma unroll
        for (int j = 0; j < 4; ++j) red[warp][cg * 4 + j] = cs[j];
      }
      __syncthreads();
      if (tid < C64_BN) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[w][tid];
        part[static_cast<size_t>(blk) * np + nt * C64_BN + tid] = s;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) rowacc[i] = fma(acc[i][j], acc[i][j], rowacc[i]);
    }
  }

  if (mode == 1) {
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double s = rowacc[i];
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      mx = valid[i] ? fmax(mx, s) : mx;
    }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    __syncthreads();
    if (lane == 0) red[0][warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double m = 0.0;
      for (int w = 0; w < 8; ++w) m = fmax(m, red[0][w]);
      part[blk] = m;
    }
  }
}

// Rows [row0, row0 + rows) of the convolution matrix A(L) (conv_op.cpp:35-46),
// column-major with leading dimension ld, written at out + off:
//   out[off + i + ld * s] = L[(v - s) mod dims],  v = row0 + i (natural order).
__global__ void icnnm_im2col64(int H, int W, int T, int kh, int kw, int kt, int64_t row0,
                               int rows, const double* __restrict__ L, double* __restrict__ out,
                               int64_t ld, int64_t off) {
  const int s = blockIdx.y;
  const int st = s % kt, q = s / kt, sw = q % kw, sh = q / kw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    const int64_t v = row0 + i;
    const int t = static_cast<int>(v % T);
    const int64_t r = v / T;
    const int w = static_cast<int>(r % W), h = static_cast<int>(r / W);
    const int hs = wrap64(h - sh, H), ws = wrap64(w - sw, W), ts = wrap64(t - st, T);
    out[off + i + ld * s] = L[(static_cast<int64_t>(hs) * W + ws) * T + ts];
  }
}

// Zero the strictly lower triangle of the leading k x k block (ld rows).
__global__ void icnnm_keep_upper(int k, int64_t ld, double* __restrict__ A) {
  const int c = blockIdx.x;
  for (int r = c + 1 + threadIdx.x; r < k; r += blockDim.x) A[r + ld * c] = 0.0;
}

// C[M x N] = A^T B with A (K x M), B (K x N), C (M x N), all column-major,
// fp64.  64 x 64 tiles, 256 threads with 4 x 4 micro-tiles.
__global__ void __launch_bounds__(256)
icnnm_dgemm_tn(int M, int N, int K, const double* __restrict__ A, const double* __restrict__ B,
               double* __restrict__ C) {
  __shared__ double As[16][65];
  __shared__ double Bs[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e & 15, c = e >> 4;
      const int gk = k0 + kk;
      As[kk][c] = (gk < K && m0 + c < M) ? A[static_cast<size_t>(m0 + c) * K + gk] : 0.0;
      Bs[kk][c] = (gk < K && n0 + c < N) ? B[static_cast<size_t>(n0 + c) * K + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tx + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][ty + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = m0 + tx + 16 * i, c = n0 + ty + 16 * j;
      if (r < M && c < N) C[static_cast<size_t>(c) * M + r] = acc[i][j];
    }
}

}  // namespace icnnm_dev

namespace icnnm_host {

using icnnm_dev::C64_BK;
using icnnm_dev::C64_BN;

// fp64 implicit GEMM out = A(L0) B over one resident copy of L0.
struct Conv64 {
  Problem p;
  Geo g;
  int64_t nb = 0;
  DBuf<double> dL;
  cudaStream_t s = 0;

  Conv64(const Problem& prob, const double* L0) : p(prob) {
    g = make_geo(p, p.dims[0], true);
    g.ktp = static_cast<int>(roundup(p.k, C64_BK));
    nb = n_bricks(g);
    check_smem(smem());
    static thread_local int done_dev = -1;
    int dev;
    CK(cudaGetDevice(&dev));
    if (done_dev != dev) {
      int optin = 0;
      CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      cudaFuncAttributes a;
      CK(cudaFuncGetAttributes(&a, icnnm_dev::icnnm_conv64));
      CK(cudaFuncSetAttribute(icnnm_dev::icnnm_conv64, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - static_cast<int>(a.sharedSizeBytes)));
      done_dev = dev;
    }
    dL.alloc(p.m);
    CK(cudaMemcpy(dL.p, L0, dL.bytes(), cudaMemcpyHostToDevice));
  }
  size_t smem() const {
    return 2 * C64_BK * C64_BN * sizeof(double) + ((g.ktp + 1) & ~1) * sizeof(int) +
           static_cast<size_t>(g.HH) * g.HW * g.HT * sizeof(double);
  }
  // Bcm: k x n column-major basis (column c = one kernel over the box).
  void launch(const double* Bcm, int n, int mode, DBuf<double>& part, int& np) {
    np = static_cast<int>(roundup(std::max(n, 1), C64_BN));
    std::vector<double> Bp(static_cast<size_t>(g.ktp) * np, 0.0);
    for (int c = 0; c < n; ++c)
      for (int s2 = 0; s2 < p.k; ++s2)
        Bp[static_cast<size_t>(s2) * np + c] = Bcm[static_cast<size_t>(c) * p.k + s2];
    DBuf<double> dB(Bp.size());
    CK(cudaMemcpy(dB.p, Bp.data(), dB.bytes(), cudaMemcpyHostToDevice));
    part.alloc(mode == 0 ? static_cast<size_t>(nb) * np : static_cast<size_t>(nb));
    icnnm_dev::icnnm_conv64<<<static_cast<unsigned>(nb), 256, smem(), s>>>(g, np, dL.p, dB.p,
                                                                          part.p, mode);
    CKL();
    CK(cudaStreamSynchronize(s));
  }
  // ||A(L0) B_c||^2 for every column c (deterministic fixed-order brick sum).
  std::vector<double> colnorm2(const double* Bcm, int n) {
    DBuf<double> part;
    int np = 0;
    launch(Bcm, n, 0, part, np);
    DBuf<double> dn(np);
    CK(cudaMemset(dn.p, 0, dn.bytes()));
    icnnm_dev::icnnm_gram_reduce<<<grid_for(np, 256), 256, 0, s>>>(np, static_cast<int>(nb),
                                                                   part.p, dn.p);
    CKL();
    std::vector<double> out(np);
    CK(cudaMemcpy(out.data(), dn.p, dn.bytes(), cudaMemcpyDeviceToHost));
    out.resize(n);
    return out;
  }
  // max over voxels v of sum_c (A(L0) B)[v, c]^2
  double rowmax(const double* Bcm, int n) {
    DBuf<double> part;
    int np = 0;
    launch(Bcm, n, 1, part, np);
    std::vector<double> h(nb);
    CK(cudaMemcpy(h.data(), part.p, part.bytes(), cudaMemcpyDeviceToHost));
    double m = 0.0;
    for (double v : h) m = std::max(m, v);
    return m;
  }
};

// C (M x N) = A^T B on the device (host arrays, column-major).
std::vector<double> dgemm_tn(int M, int N, int K, const double* A, const double* B) {
  DBuf<double> dA(static_cast<size_t>(K) * M), dB(static_cast<size_t>(K) * N),
      dC(static_cast<size_t>(M) * N);
  CK(cudaMemcpy(dA.p, A, dA.bytes(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB.p, B, dB.bytes(), cudaMemcpyHostToDevice));
  dim3 grid((M + 63) / 64, (N + 63) / 64);
  icnnm_dev::icnnm_dgemm_tn<<<grid, 256>>>(M, N, K, dA.p, dB.p, dC.p);
  CKL();
  std::vector<double> C(static_cast<size_t>(M) * N);
  CK(cudaMemcpy(C.data(), dC.p, dC.bytes(), cudaMemcpyDeviceToHost));
  return C;
}

// support_from (analysis.cpp:40-49)
std::vector<int64_t> support_from(const std::vector<double>& sigma, double rank_tol) {
  std::vector<int64_t> sup;
  double smax = 0.0;
  for (double v : sigma) smax = std::max(smax, v);
  if (smax == 0) return sup;
  for (size_t i = 0; i < sigma.size(); ++i)
    if (sigma[i] > rank_tol * smax) sup.push_back(static_cast<int64_t>(i));
  return sup;
}

// power_iteration_top_eig (analysis.cpp:51-69); S is n x n symmetric.  S*w
// of one iteration is S*v of the next (v <- w), so it is computed once.
double power_iteration_top_eig(const std::vector<double>& S, int n) {
  auto matvec = [&](const std::vector<double>& x, std::vector<double>& y) {
    for (int i = 0; i < n; ++i) y[i] = 0.0;
    for (int c = 0; c < n; ++c) {
      const double xc = x[c];
      const double* col = S.data() + static_cast<size_t>(c) * n;
      for (int i = 0; i < n; ++i) y[i] += col[i] * xc;
    }
  };
  std::vector<double> v(n, 1.0 / std::sqrt(static_cast<double>(n))), w(n), Sv(n), Sw(n);
  matvec(v, Sv);
  double eig = 0;
  for (int it = 0; it < 10000; ++it) {
    w = Sv;
    double nw = 0;
    for (double x : w) nw += x * x;
    nw = std::sqrt(nw);
    if (nw == 0) return 0;
    for (double& x : w) x /= nw;
    matvec(w, Sw);
    double ne = 0;
    for (int i = 0; i < n; ++i) ne += w[i] * Sw[i];
    const bool done = std::abs(ne - eig) <= 1e-10 * std::max(1.0, std::abs(ne));
    eig = ne;
    v.swap(w);
    Sv.swap(Sw);
    if (done && it > 0) break;
  }
  return eig;
}

double tensor_norm2(const Problem& p, const double* L0) {
  double s = 0;
  for (int64_t i = 0; i < p.m; ++i) s += L0[i] * L0[i];
  return s;
}

// conv_gram of L0 (spectral.cpp:62-79) from the fp64 lag kernel.
std::vector<double> conv_gram_host(const Problem& p, const double* dL0) {
  const size_t nl = static_cast<size_t>(2 * p.kd[0] - 1) * (2 * p.kd[1] - 1) * (2 * p.kd[2] - 1);
  DBuf<double> dR(nl);
  CK(cudaMemset(dR.p, 0, dR.bytes()));
  set_smem_attrs();
  gram_lags_accumulate(p, dL0, dR.p, 0);
  std::vector<double> R(nl), G(static_cast<size_t>(p.k) * p.k);
  CK(cudaMemcpy(R.data(), dR.p, dR.bytes(), cudaMemcpyDeviceToHost));
  gram_from_lags(p, R, G.data());
  return G;
}

// spectral_corr_coeff body (analysis.cpp:79-96) given sigma and its support.
double alpha_from(const Problem& p, const std::vector<double>& G, const double* K,
                  const std::vector<double>& sigma, const std::vector<int64_t>& sup) {
  const int k = p.k, r = static_cast<int>(sup.size());
  std::vector<double> KD(static_cast<size_t>(k) * r);
  for (int j = 0; j < r; ++j) {
    const double* src = K + static_cast<size_t>(sup[j]) * k;
    const double d = sigma[sup[j]];
    for (int s2 = 0; s2 < k; ++s2) KD[static_cast<size_t>(j) * k + s2] = src[s2] / d;
  }
  std::vector<double> T = dgemm_tn(k, r, k, G.data(), KD.data());  // G^T KD = G KD
  std::vector<double> S = dgemm_tn(r, r, k, KD.data(), T.data());  // KD^T (G KD)
  return std::sqrt(std::max(0.0, power_iteration_top_eig(S, r)));
}

#define CKS(x)                                                                     \
  do {                                                                             \
    cusolverStatus_t st_ = (x);                                                    \
    if (st_ != CUSOLVER_STATUS_SUCCESS)                                            \
      ::icnnm_host::fail(ICNNM_CUDA_ERROR, std::string(#x) + ": cusolver status " + \
                                               std::to_string(static_cast<int>(st_)));  \
  } while (0)

struct Cusolver {
  cusolverDnHandle_t h = nullptr;
  Cusolver() { CKS(cusolverDnCreate(&h)); }
  ~Cusolver() {
    if (h) cusolverDnDestroy(h);
  }
};

// Singular values (descending) and right singular vectors V (k x k,
// column-major, column i <-> s[i]) of the m x k convolution matrix A(L0):
// streaming TSQR  [R; A_b] = Q R'  over row blocks A_b gathered on the GPU,
// then the SVD of the final R.  Device memory: (k + rows_b) x k doubles.
void conv_svd(const Problem& p, const double* dL0, std::vector<double>& s,
              std::vector<double>& V) {
  const int k = p.k;
  const int64_t m = p.m;
  const int64_t budget_rows = std::max<int64_t>(4 * k, (int64_t(1) << 28) / k);  // 2 GB
  const int rows_b = static_cast<int>(std::min<int64_t>(m, budget_rows));
  const int64_t ld = static_cast<int64_t>(k) + rows_b;
  if (ld > (int64_t(1) << 31) - 1) invalid("conv_coherence: block too large");
  Cusolver cs;
  DBuf<double> Wb(static_cast<size_t>(ld) * k), tau(k);
  DBuf<int> info(1);
  int lwork = 0;
  CKS(cusolverDnDgeqrf_bufferSize(cs.h, static_cast<int>(ld), k, Wb.p, static_cast<int>(ld),
                                  &lwork));
  DBuf<double> work(std::max(lwork, 1));
  CK(cudaMemset(Wb.p, 0, Wb.bytes()));  // R_0 = 0
  const int H = static_cast<int>(p.dims[0]), W = static_cast<int>(p.dims[1]),
            T = static_cast<int>(p.dims[2]);
  for (int64_t row0 = 0; row0 < m; row0 += rows_b) {
    const int rows = static_cast<int>(std::min<int64_t>(rows_b, m - row0));
    if (rows < rows_b)  // last partial block: zero rows contribute nothing
      CK(cudaMemset2D(Wb.p + k + rows, sizeof(double) * ld, 0, sizeof(double) * (rows_b - rows),
                      k));
    dim3 grid(static_cast<unsigned>(std::min<int64_t>((rows + 255) / 256, 4096)),
              static_cast<unsigned>(k));
    icnnm_dev::icnnm_im2col64<<<grid, 256>>>(H, W, T, static_cast<int>(p.kd[0]),
                                             static_cast<int>(p.kd[1]), static_cast<int>(p.kd[2]),
                                             row0, rows, dL0, Wb.p, ld, k);
    CKL();
    CKS(cusolverDnDgeqrf(cs.h, static_cast<int>(ld), k, Wb.p, static_cast<int>(ld), tau.p,
                         work.p, lwork, info.p));
    icnnm_dev::icnnm_keep_upper<<<k, 128>>>(k, ld, Wb.p);
    CKL();
  }
  int hinfo = 0;
  CK(cudaMemcpy(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (hinfo != 0) fail(ICNNM_RUNTIME_ERROR, "conv_coherence: QR failed");
  // SVD of R (k x k, leading block of Wb).
  DBuf<double> R(static_cast<size_t>(k) * k), S(k), VT(static_cast<size_t>(k) * k);
  CK(cudaMemcpy2D(R.p, sizeof(double) * k, Wb.p, sizeof(double) * ld, sizeof(double) * k, k,
                  cudaMemcpyDeviceToDevice));
  int lw2 = 0;
  CKS(cusolverDnDgesvd_bufferSize(cs.h, k, k, &lw2));
  DBuf<double> work2(std::max(lw2, 1)), rwork(k);
  CKS(cusolverDnDgesvd(cs.h, 'N', 'A', k, k, R.p, k, S.p, nullptr, 1, VT.p, k, work2.p, lw2,
                       rwork.p, info.p));
  CK(cudaMemcpy(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (hinfo != 0) fail(ICNNM_RUNTIME_ERROR, "conv_coherence: SVD did not converge");
  s.resize(k);
  std::vector<double> vt(static_cast<size_t>(k) * k);
  CK(cudaMemcpy(s.data(), S.p, S.bytes(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(vt.data(), VT.p, VT.bytes(), cudaMemcpyDeviceToHost));
  V.assign(static_cast<size_t>(k) * k, 0.0);
  for (int i = 0; i < k; ++i)      // V[:, i] = row i of VT
    for (int j = 0; j < k; ++j) V[static_cast<size_t>(i) * k + j] = vt[i + static_cast<size_t>(k) * j];
}

void conv_coherence_impl(const Problem& p, const double* L0, Conv64& conv, double rank_tol,
                         icnnm_conv_coherence* out) {
  if (tensor_norm2(p, L0) == 0) invalid("conv_coherence: zero tensor");
  const int k = p.k;
  std::vector<double> s, V;
  conv_svd(p, conv.dL.p, s, V);
  int r = 0;
  for (int i = 0; i < k; ++i)
    if (s[i] > rank_tol * s[0]) ++r;
  if (r == 0) invalid("conv_coherence: zero tensor");
  double vmax = 0;
  for (int j = 0; j < k; ++j) {
    double acc = 0;
    for (int i = 0; i < r; ++i) {
      const double v = V[static_cast<size_t>(i) * k + j];
      acc += v * v;
    }
    vmax = std::max(vmax, acc);
  }
  std::vector<double> Us(static_cast<size_t>(k) * r);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < k; ++j)
      Us[static_cast<size_t>(i) * k + j] = V[static_cast<size_t>(i) * k + j] / s[i];
  const double umax = conv.rowmax(Us.data(), r);
  out->rank = r;
  out->mu1 = static_cast<double>(p.m) / r * umax;
  out->mu2 = static_cast<double>(k) / r * vmax;
  out->tau = s[0] / s[r - 1];
}

void thresholds_impl(const icnnm_threshold_inputs& in, icnnm_threshold_values* t) {
  // thresholds (analysis.cpp:137-153)
  const double a2 = in.alpha_K * in.alpha_K;
  const double k = static_cast<double>(in.k), m = static_cast<double>(in.m);
  const double rk = static_cast<double>(in.r_K), r0 = static_cast<double>(in.r0);
  t->rho_min_noiseless = 1.0 - k / ((1.0 + a2) * in.mu_K_I * rk * m);
  t->rho_min_noisy = 1.0 - 0.64 * k / ((0.64 + a2) * in.mu_K_I * rk * m);
  t->error_bound_factor =
      (18.0 * std::sqrt(k) + 2.0) * (in.alpha_K + std::sqrt(1.0 + a2)) / in.alpha_K;
  t->icnnm_ideal_bound = 1.0 - 0.5 * k / (in.mu2 * r0 * m);
  t->cnnm_bound = 1.0 - 0.25 * k / (std::max(in.mu1, in.mu2) * r0 * m);
  t->certified = in.rho0 > t->rho_min_noiseless ? 1 : 0;
}

double active_coherence_impl(int64_t k, const double* K, int64_t n, const int64_t* sup) {
  // active_coherence (analysis.cpp:98-109)
  if (n <= 0) invalid("active_coherence: empty support");
  if (!K || !sup) invalid("null argument");
  for (int64_t c = 0; c < n; ++c)
    if (sup[c] < 0 || sup[c] >= k) invalid("active_coherence: support index out of range");
  double max_row = 0;
  for (int64_t r = 0; r < k; ++r) {
    double s = 0;
    for (int64_t c = 0; c < n; ++c) {
      const double v = K[static_cast<size_t>(sup[c]) * k + r];
      s += v * v;
    }
    max_row = std::max(max_row, s);
  }
  return static_cast<double>(k) / static_cast<double>(n) * max_row;
}

std::vector<double> relative_eigenvalues(const Problem& p, Conv64& conv, const double* K) {
  std::vector<double> s2 = conv.colnorm2(K, p.k);
  for (double& v : s2) v = std::sqrt(v);
  return s2;
}

void check_basis_args(const Problem& p, const double* L0, const double* K, const double* evals) {
  if (!L0 || !K) invalid("null argument");
  validate_basis(p.k, K, evals);
}

}  // namespace icnnm_host

using namespace icnnm_host;

extern "C" {

int icnnm_cuda_relative_eigenvalues(int order, const int64_t* dims, const double* L0,
                                    const int64_t* kdims, const double* K, const double* evals,
                                    int device, double* sigma) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    check_basis_args(p, L0, K, evals);
    if (!sigma) invalid("null argument");
    DeviceScope ds(device);
    Conv64 conv(p, L0);
    std::vector<double> s = relative_eigenvalues(p, conv, K);
    std::copy(s.begin(), s.end(), sigma);
  });
}

int icnnm_cuda_relative_conv_rank(int order, const int64_t* dims, const double* L0,
                                  const int64_t* kdims, const double* K, const double* evals,
                                  double rank_tol, int device, int64_t* r_K, int64_t* support) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    check_basis_args(p, L0, K, evals);
    if (!r_K) invalid("null argument");
    DeviceScope ds(device);
    Conv64 conv(p, L0);
    std::vector<int64_t> sup = support_from(relative_eigenvalues(p, conv, K), rank_tol);
    *r_K = static_cast<int64_t>(sup.size());
    if (support) std::copy(sup.begin(), sup.end(), support);
  });
}

int icnnm_cuda_spectral_corr_coeff(int order, const int64_t* dims, const double* L0,
                                   const int64_t* kdims, const double* K, const double* evals,
                                   double rank_tol, int device, double* alpha) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    check_basis_args(p, L0, K, evals);
    if (!alpha) invalid("null argument");
    DeviceScope ds(device);
    Conv64 conv(p, L0);
    std::vector<double> sigma = relative_eigenvalues(p, conv, K);
    std::vector<int64_t> sup = support_from(sigma, rank_tol);
    if (sup.empty()) invalid("spectral_corr_coeff: r_K = 0, undefined");
    *alpha = alpha_from(p, conv_gram_host(p, conv.dL.p), K, sigma, sup);
  });
}

int icnnm_active_coherence(int64_t k, const double* K, int64_t n_support, const int64_t* support,
                           double* out) {
  return guard([&] {
    if (!out) invalid("null argument");
    *out = active_coherence_impl(k, K, n_support, support);
  });
}

int icnnm_cuda_conv_coherence(int order, const int64_t* dims, const double* L0,
                              const int64_t* kdims, double rank_tol, int device,
                              icnnm_conv_coherence* out) {
  return guard([&] {
    Problem p = make_problem(order, dims, kdims);
    if (!L0 || !out) invalid("null argument");
    DeviceScope ds(device);
    if (tensor_norm2(p, L0) == 0) invalid("conv_coherence: zero tensor");
    Conv64 conv(p, L0);
    conv_coherence_impl(p, L0, conv, rank_tol, out);
  });
}

int icnnm_thresholds(const icnnm_threshold_inputs* in, icnnm_threshold_values* out) {
  return guard([&] {
    if (!in || !out) invalid("null argument");
    thresholds_impl(*in, out);
  });
}

int icnnm_cuda_analyze_recovery(int order, const int64_t* dims, const double* L0,
                                const int64_t* kdims, const double* K, const double* evals,
                                const double* mask, double rank_tol, int device,
                                icnnm_recovery_diagnostics* d) {
  return guard([&] {
    // analyze_recovery (analysis.cpp:155-185)
    Problem p = make_problem(order, dims, kdims);
    check_basis_args(p, L0, K, evals);
    if (!mask || !d) invalid("null argument");
    double msum = 0;
    for (int64_t i = 0; i < p.m; ++i) {
      if (mask[i] != 0.0 && mask[i] != 1.0) invalid("SamplingMask: entries must be 0 or 1");
      msum += mask[i];
    }
    DeviceScope ds(device);
    Conv64 conv(p, L0);
    std::vector<double> sigma = relative_eigenvalues(p, conv, K);
    std::vector<int64_t> sup = support_from(sigma, rank_tol);
    if (sup.empty()) invalid("analyze_recovery: zero target, diagnostics undefined");
    const std::vector<double> G = conv_gram_host(p, conv.dL.p);
    d->r_K = static_cast<int64_t>(sup.size());
    if (d->support_I) std::copy(sup.begin(), sup.end(), d->support_I);
    d->alpha_K = alpha_from(p, G, K, sigma, sup);
    d->mu_K_I = active_coherence_impl(p.k, K, d->r_K, sup.data());
    icnnm_conv_coherence cc{};
    conv_coherence_impl(p, L0, conv, rank_tol, &cc);
    d->mu1 = cc.mu1;
    d->mu2 = cc.mu2;
    d->tau = cc.tau;
    d->r0 = cc.rank;
    d->rho0 = static_cast<double>(static_cast<int64_t>(msum + 0.5)) / static_cast<double>(p.m);
    icnnm_threshold_inputs in{d->r_K, d->alpha_K, d->mu_K_I, d->mu1, d->mu2,
                              d->r0,  p.k,        p.m,       d->rho0};
    icnnm_threshold_values t{};
    thresholds_impl(in, &t);
    d->rho_min_noiseless = t.rho_min_noiseless;
    d->rho_min_noisy = t.rho_min_noisy;
    d->error_bound_factor = t.error_bound_factor;
    d->cnnm_bound = t.cnnm_bound;
    d->icnnm_ideal_bound = t.icnnm_ideal_bound;
    d->certified = t.certified;
  });
}

}  // extern "C"
