// CNNM baseline on the GPU: cnnm_solve
// (/root/reference/proj/core/src/solver.cpp:161-170) = the shared ADMM loop
// (:62-146) with K = I and the singular-value-thresholding Z-update
// svt(W, tau) (:52-57).
//
// The reference runs an Eigen BDCSVD of the m x k matrix every iteration.
// Here, per iteration, in fp64:
//   G = Wa^T Wa                     cuBLAS DSYRK (m x k -> k x k)
//   G = V diag(lambda) V^T          cuSOLVER syevd (k x k)
//   P = V diag(f) V^T, f = max(sqrt(lambda) - tau, 0) / sqrt(lambda)
//   Z = Wa P                        cuBLAS DGEMM  (= U max(S - tau, 0) V^T)
// and three fused bandwidth kernels for the rest of the loop body: the
// adjoint gather + L update (cnnm_update), the multiplier update fused with
// the next iteration's Wa = A(L) - Y/theta (cnnm_dual), and the shrink
// factors.  With K = I the forward "GEMM" A(L)K is a gather of L, so A(L) is
// never stored: it is recomputed from L (L2-resident) inside the kernels.
//
// SVT through the Gram: directions whose singular value is below the fp64
// Gram resolution (~1e-8 s_max) carry Wa-components of that size, so the
// error this adds to Z is bounded by ~1e-8 ||Wa||.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <vector>

#include "icnnm_host_common.h"

namespace icnnm_dev {

__device__ __forceinline__ int wrapc(int x, int n) {
  int r = x % n;
  return r < 0 ? r + n : r;
}

struct CGeo {
  int H, W, T, kh, kw, kt;
  int64_t m;
  int k;
};

__device__ __forceinline__ void tap_of(const CGeo& g, int s, int& sh, int& sw, int& st) {
  st = s % g.kt;
  const int q = s / g.kt;
  sw = q % g.kw;
  sh = q / g.kw;
}

// Flat index of voxel v shifted by sign * (sh, sw, st), periodic.
__device__ __forceinline__ int64_t shifted(const CGeo& g, int64_t v, int sh, int sw, int st,
                                           int sign) {
  const int t = static_cast<int>(v % g.T);
  const int64_t r = v / g.T;
  const int w = static_cast<int>(r % g.W), h = static_cast<int>(r / g.W);
  const int hs = wrapc(h + sign * sh, g.H), ws = wrapc(w + sign * sw, g.W),
            ts = wrapc(t + sign * st, g.T);
  return (static_cast<int64_t>(hs) * g.W + ws) * g.T + ts;
}

// Wa[i + m s] = L[(i - s) mod dims] - Y[i + m s] / theta   (Y == nullptr: 0)
__global__ void __launch_bounds__(256)
cnnm_prep(CGeo g, const double* __restrict__ L, const double* __restrict__ Y, double inv_theta,
          double* __restrict__ Wa) {
  const int s = blockIdx.y;
  int sh, sw, st;
  tap_of(g, s, sh, sw, st);
  const size_t col = static_cast<size_t>(g.m) * s;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double akl = L[shifted(g, i, sh, sw, st, -1)];
    Wa[col + i] = Y ? akl - Y[col + i] * inv_theta : akl;
  }
}

// Block sum of NV values into part[blockIdx.x * stride + j*?]; helper.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* out /* NV slots */) {
  __shared__ double sh[NV][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double x = v[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sh[j][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double x = threadIdx.x < nw ? sh[j][threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (threadIdx.x == 0) out[j] = x;
    }
  }
}

// adj[i] = sum_s (Y + theta Z)[(i + s) mod dims, s]            (conv_op.cpp:57-77)
// L[i]  <- (adj/k + lambda pm[i]) / (lambda mask[i] + theta)   (solver.cpp:110-116)
// part[blockIdx.x * 3 + {0,1,2}] = sum (L_new - L)^2, sum L^2, sum (mask L_new - pm)^2
__global__ void __launch_bounds__(256)
cnnm_update(CGeo g, const double* __restrict__ Y, const double* __restrict__ Z, double theta,
            double lambda, const double* __restrict__ pm, const double* __restrict__ mask,
            double* __restrict__ L, double* __restrict__ part) {
  double acc[3] = {0.0, 0.0, 0.0};
  const double inv_k = 1.0 / static_cast<double>(g.k);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double adj = 0.0;
    for (int s = 0; s < g.k; ++s) {
      int sh, sw, st;
      tap_of(g, s, sh, sw, st);
      const size_t idx = static_cast<size_t>(g.m) * s + shifted(g, i, sh, sw, st, +1);
      adj += Y[idx] + theta * Z[idx];
    }
    const double mk = mask[i], p = pm[i];
    const double lnew = (adj * inv_k + lambda * p) / (lambda * mk + theta);
    const double lold = L[i];
    const double d = lnew - lold, f = lnew * mk - p;
    acc[0] += d * d;
    acc[1] += lold * lold;
    acc[2] += f * f;
    L[i] = lnew;
  }
  block_sum<3>(acc, part + blockIdx.x * 3);
}

// gap = Z - A(L); Y += theta gap; Wa = A(L) - Y/theta_next   (solver.cpp:121-126, :108)
// part_gap[bx * k + s] = sum gap^2, part_zn[bx * k + s] = sum Z^2 over the block's rows.
__global__ void __launch_bounds__(256)
cnnm_dual(CGeo g, const double* __restrict__ L, const double* __restrict__ Z,
          double* __restrict__ Y, double theta, double inv_theta_next, double* __restrict__ Wa,
          double* __restrict__ part_gap, double* __restrict__ part_zn) {
  const int s = blockIdx.y;
  int sh, sw, st;
  tap_of(g, s, sh, sw, st);
  const size_t col = static_cast<size_t>(g.m) * s;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double akl = L[shifted(g, i, sh, sw, st, -1)];
    const double z = Z[col + i];
    const double gap = z - akl;
    const double y = Y[col + i] + theta * gap;
    Y[col + i] = y;
    Wa[col + i] = akl - y * inv_theta_next;
    acc[0] += gap * gap;
    acc[1] += z * z;
  }
  double out[2];
  block_sum<2>(acc, out);
  if (threadIdx.x == 0) {
    part_gap[static_cast<size_t>(blockIdx.x) * g.k + s] = out[0];
    part_zn[static_cast<size_t>(blockIdx.x) * g.k + s] = out[1];
  }
}

// Vf[:, c] = V[:, c] * max(s_c - tau, 0) / s_c,  s_c = sqrt(max(lambda_c, 0))
__global__ void cnnm_shrink(int k, const double* __restrict__ V, const double* __restrict__ lam,
                            double tau, double* __restrict__ Vf) {
  const int c = blockIdx.x;
  const double sv = sqrt(fmax(lam[c], 0.0));
  const double f = sv > tau ? (sv - tau) / sv : 0.0;
  for (int r = threadIdx.x; r < k; r += blockDim.x)
    Vf[static_cast<size_t>(c) * k + r] = V[static_cast<size_t>(c) * k + r] * f;
}

// ---------------------------------------------------------------------------
// FP64 engine of icnnm_solve (ICNNM_ENGINE_F64): the literal loop
// (solver.cpp:107-139) with the three m x k matrices Wa/AKL, Z, Y in fp64 and
// the two contractions as cuBLAS DGEMMs.  Not the hot path: it exists so that
// tolerances below the fp32 engines' resolution (the reference's defaults
// tol_primal = 1e-7, tol_change = 1e-8) stop the loop where the reference does.
// ---------------------------------------------------------------------------
// pm = M mask; L = pm (+ (1 - mask) mean)                      (solver.cpp:80-86)
__global__ void __launch_bounds__(256)
f64_init(int64_t m, const double* __restrict__ M, const double* __restrict__ mask, int mean_fill,
         double mean, double* __restrict__ pm, double* __restrict__ L) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double mk = mask[i], p = M[i] * mk;
    pm[i] = p;
    L[i] = mean_fill ? p + (1.0 - mk) * mean : p;
  }
}

// out = Y + theta Z                                             (solver.cpp:110 operand)
__global__ void __launch_bounds__(256)
f64_ypz(int64_t n, const double* __restrict__ Y, const double* __restrict__ Z, double theta,
        double* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = Y[i] + theta * Z[i];
}

// adj[i] = sum_s WK[(i + s) mod dims, s]                        (conv_op.cpp:57-77)
// L[i]  <- (adj/k + lambda pm[i]) / (lambda mask[i] + theta)    (solver.cpp:112-116)
// part[blockIdx.x * 3 + {0,1,2}] = sum (L_new - L)^2, sum L^2, sum (mask L_new - pm)^2
__global__ void __launch_bounds__(256)
f64_update(CGeo g, const double* __restrict__ WK, double theta, double lambda,
           const double* __restrict__ pm, const double* __restrict__ mask,
           double* __restrict__ L, double* __restrict__ part) {
  double acc[3] = {0.0, 0.0, 0.0};
  const double inv_k = 1.0 / static_cast<double>(g.k);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double adj = 0.0;
    for (int s = 0; s < g.k; ++s) {
      int sh, sw, st;
      tap_of(g, s, sh, sw, st);
      adj += WK[static_cast<size_t>(g.m) * s + shifted(g, i, sh, sw, st, +1)];
    }
    const double mk = mask[i], p = pm[i];
    const double lnew = (adj * inv_k + lambda * p) / (lambda * mk + theta);
    const double lold = L[i];
    const double d = lnew - lold, f = lnew * mk - p;
    acc[0] += d * d;
    acc[1] += lold * lold;
    acc[2] += f * f;
    L[i] = lnew;
  }
  block_sum<3>(acc, part + blockIdx.x * 3);
}

// gap = Z - AKL; Y += theta gap; Wa = AKL - Y/theta_next (in place of AKL)
// (solver.cpp:123-126, :108); per-block column partials of gap^2 and Z^2
__global__ void __launch_bounds__(256)
f64_dual(int64_t m, int k, const double* __restrict__ Z, double* __restrict__ Y, double theta,
         double inv_theta_next, double* __restrict__ Wa, double* __restrict__ part_gap,
         double* __restrict__ part_zn) {
  const int s = blockIdx.y;
  const size_t col = static_cast<size_t>(m) * s;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double akl = Wa[col + i];
    const double z = Z[col + i];
    const double gap = z - akl;
    const double y = Y[col + i] + theta * gap;
    Y[col + i] = y;
    Wa[col + i] = akl - y * inv_theta_next;
    acc[0] += gap * gap;
    acc[1] += z * z;
  }
  double out[2];
  block_sum<2>(acc, out);
  if (threadIdx.x == 0) {
    part_gap[static_cast<size_t>(blockIdx.x) * k + s] = out[0];
    part_zn[static_cast<size_t>(blockIdx.x) * k + s] = out[1];
  }
}

}  // namespace icnnm_dev

namespace icnnm_host {

void validate_cfg(const icnnm_solver_config* c);

#define CKB(x)                                                                         \
  do {                                                                                 \
    cublasStatus_t st_ = (x);                                                          \
    if (st_ != CUBLAS_STATUS_SUCCESS)                                                  \
      ::icnnm_host::fail(ICNNM_CUDA_ERROR,                                             \
                         std::string(#x) + ": cublas status " + std::to_string(static_cast<int>(st_))); \
  } while (0)
#define CKS2(x)                                                                        \
  do {                                                                                 \
    cusolverStatus_t st_ = (x);                                                        \
    if (st_ != CUSOLVER_STATUS_SUCCESS)                                                \
      ::icnnm_host::fail(ICNNM_CUDA_ERROR, std::string(#x) + ": cusolver status " +   \
                                               std::to_string(static_cast<int>(st_))); \
  } while (0)

struct CnnmHandles {
  cudaStream_t s = nullptr;
  cublasHandle_t b = nullptr;
  cusolverDnHandle_t q = nullptr;
  CnnmHandles() {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CKB(cublasCreate(&b));
    CKB(cublasSetStream(b, s));
    CKS2(cusolverDnCreate(&q));
    CKS2(cusolverDnSetStream(q, s));
  }
  ~CnnmHandles() {
    if (q) cusolverDnDestroy(q);
    if (b) cublasDestroy(b);
    if (s) cudaStreamDestroy(s);
  }
};

void cnnm_solve_impl(const Problem& p, const double* M, const double* mask,
                     const icnnm_solver_config& cfg, double* L_out, icnnm_solve_report* rep) {
  const auto t_start = std::chrono::steady_clock::now();
  const int64_t m = p.m;
  const int k = p.k;
  const double kd = static_cast<double>(k);
  // admm_solve setup (solver.cpp:78-102)
  std::vector<double> pm(m), L(m);
  double amax = 0, n2 = 0, sum = 0;
  int64_t obs = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (mask[i] != 0.0 && mask[i] != 1.0) invalid("SamplingMask: entries must be 0 or 1");
  }
  for (int64_t i = 0; i < m; ++i) obs += mask[i] == 1.0;
  if (obs == 0) invalid("solve: empty sampling set");
  for (int64_t i = 0; i < m; ++i)
    if (!std::isfinite(M[i])) invalid("solve: observations: non-finite tensor entries");
  for (int64_t i = 0; i < m; ++i) {
    pm[i] = M[i] * mask[i];
    amax = std::max(amax, std::fabs(pm[i]));
    n2 += pm[i] * pm[i];
    sum += pm[i];
  }
  for (int64_t i = 0; i < m; ++i) L[i] = pm[i];
  if (cfg.init_fill == ICNNM_INIT_MEAN) {
    const double mean = sum / static_cast<double>(obs);
    for (int64_t i = 0; i < m; ++i) L[i] += (1.0 - mask[i]) * mean;
  }
  double theta = cfg.has_theta0 ? cfg.theta0 : 1e-2 * amax * kd;
  if (theta <= 0) theta = 1e-2;
  theta = std::min(theta, cfg.theta_max);
  double res_scale = std::sqrt(kd) * std::sqrt(n2);
  if (res_scale == 0) res_scale = 1.0;

  CnnmHandles hd;
  const size_t mk = static_cast<size_t>(m) * k;
  DBuf<double> dL(m), dpm(m), dmask(m), Y(mk), Wa(mk), Z(mk), G(static_cast<size_t>(k) * k),
      Vf(static_cast<size_t>(k) * k), P(static_cast<size_t>(k) * k), lam(k);
  DBuf<int> info(1);
  CK(cudaMemcpyAsync(dL.p, L.data(), dL.bytes(), cudaMemcpyHostToDevice, hd.s));
  CK(cudaMemcpyAsync(dpm.p, pm.data(), dpm.bytes(), cudaMemcpyHostToDevice, hd.s));
  CK(cudaMemcpyAsync(dmask.p, mask, dmask.bytes(), cudaMemcpyHostToDevice, hd.s));
  CK(cudaMemsetAsync(Y.p, 0, Y.bytes(), hd.s));
  int lwork = 0;
  CKS2(cusolverDnDsyevd_bufferSize(hd.q, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, G.p,
                                   k, lam.p, &lwork));
  DBuf<double> work(std::max(lwork, 1));

  icnnm_dev::CGeo g{static_cast<int>(p.dims[0]), static_cast<int>(p.dims[1]),
                    static_cast<int>(p.dims[2]), static_cast<int>(p.kd[0]),
                    static_cast<int>(p.kd[1]), static_cast<int>(p.kd[2]), m, k};
  const int gx_up = static_cast<int>(std::min<int64_t>((m + 255) / 256, 592));
  const int gx_col = static_cast<int>(std::min<int64_t>((m + 255) / 256, 64));
  DBuf<double> part_up(static_cast<size_t>(gx_up) * 3), part_gap(static_cast<size_t>(gx_col) * k),
      part_zn(static_cast<size_t>(gx_col) * k), red(2 * static_cast<size_t>(k));
  std::vector<double> hup(static_cast<size_t>(gx_up) * 3), hred(2 * static_cast<size_t>(k));

  icnnm_dev::cnnm_prep<<<dim3(gx_col, k), 256, 0, hd.s>>>(g, dL.p, nullptr, 0.0, Wa.p);
  CKL();

  const double one = 1.0, zero = 0.0;
  rep->iterations = 0;
  rep->termination = ICNNM_TERM_MAX_ITERS;
  const auto t_loop = std::chrono::steady_clock::now();
  for (int it = 0; it < cfg.max_iters; ++it) {
    const double tau = 1.0 / theta;
    // Z = svt(Wa, 1/theta)                                         (solver.cpp:108, :52-57)
    CKB(cublasDsyrk(hd.b, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, k, static_cast<int>(m), &one,
                    Wa.p, static_cast<int>(m), &zero, G.p, k));
    CKS2(cusolverDnDsyevd(hd.q, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, G.p, k,
                          lam.p, work.p, lwork, info.p));
    icnnm_dev::cnnm_shrink<<<k, 128, 0, hd.s>>>(k, G.p, lam.p, tau, Vf.p);
    CKL();
    CKB(cublasDgemm(hd.b, CUBLAS_OP_N, CUBLAS_OP_T, k, k, k, &one, Vf.p, k, G.p, k, &zero, P.p,
                    k));
    CKB(cublasDgemm(hd.b, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(m), k, k, &one, Wa.p,
                    static_cast<int>(m), P.p, k, &zero, Z.p, static_cast<int>(m)));
    // L update (:110-120)
    icnnm_dev::cnnm_update<<<gx_up, 256, 0, hd.s>>>(g, Y.p, Z.p, theta, cfg.lambda, dpm.p,
                                                     dmask.p, dL.p, part_up.p);
    CKL();
    const double theta_next = std::min(theta * cfg.theta_growth, cfg.theta_max);
    // gap, Y update (:121-126) and the next iteration's Wa
    icnnm_dev::cnnm_dual<<<dim3(gx_col, k), 256, 0, hd.s>>>(g, dL.p, Z.p, Y.p, theta,
                                                            1.0 / theta_next, Wa.p, part_gap.p,
                                                            part_zn.p);
    CKL();
    CK(cudaMemsetAsync(red.p, 0, red.bytes(), hd.s));
    icnnm_dev::icnnm_gram_reduce<<<grid_for(k, 256), 256, 0, hd.s>>>(k, gx_col, part_gap.p,
                                                                     red.p);
    icnnm_dev::icnnm_gram_reduce<<<grid_for(k, 256), 256, 0, hd.s>>>(k, gx_col, part_zn.p,
                                                                     red.p + k);
    CKL();
    CK(cudaMemcpyAsync(hup.data(), part_up.p, part_up.bytes(), cudaMemcpyDeviceToHost, hd.s));
    CK(cudaMemcpyAsync(hred.data(), red.p, red.bytes(), cudaMemcpyDeviceToHost, hd.s));
    CK(cudaStreamSynchronize(hd.s));
    double dl2 = 0, l2o = 0, fit = 0, gap2 = 0, col_sum = 0;
    for (int b = 0; b < gx_up; ++b) {
      dl2 += hup[3 * b];
      l2o += hup[3 * b + 1];
      fit += hup[3 * b + 2];
    }
    for (int c = 0; c < k; ++c) {
      gap2 += hred[c];
      col_sum += std::sqrt(hred[k + c]);
    }
    const double l_change = std::sqrt(dl2) / std::max(std::sqrt(l2o), 1e-300);
    const double residual = std::sqrt(gap2) / res_scale;
    theta = theta_next;
    if (rep->objective) rep->objective[it] = col_sum + 0.5 * cfg.lambda * kd * fit;
    if (rep->primal_residual) rep->primal_residual[it] = residual;
    if (rep->l_change) rep->l_change[it] = l_change;
    rep->iterations = it + 1;
    if (residual < cfg.tol_primal || l_change < cfg.tol_change) {  // :136-139
      rep->termination = ICNNM_TERM_CONVERGED;
      break;
    }
  }
  int hinfo = 0;
  CK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, hd.s));
  CK(cudaMemcpyAsync(L_out, dL.p, dL.bytes(), cudaMemcpyDeviceToHost, hd.s));
  CK(cudaStreamSynchronize(hd.s));
  if (hinfo != 0) fail(ICNNM_RUNTIME_ERROR, "cnnm_solve: eigensolver did not converge");
  const auto t_end = std::chrono::steady_clock::now();
  rep->loop_seconds = std::chrono::duration<double>(t_end - t_loop).count();
  rep->device_seconds = rep->loop_seconds;
  rep->wall_time_seconds = std::chrono::duration<double>(t_end - t_start).count();
}

// FP64 engine (see the kernels above).  dM / dmask: the staged problem on the
// device (validated at upload); dL receives the iterate.  The theta schedule
// and the stopping test are the reference's (solver.cpp:88-91, :126, :136-139),
// evaluated on the host once per iteration (one small D2H, off the hot path).
void icnnm_f64_loop(const Problem& p, const double* dM, const double* dmask,
                    const double* K_colmajor, const icnnm_solver_config& cfg, double pm_absmax,
                    double pm_norm2, double pm_sum, int64_t observed, double* dL,
                    std::vector<icnnm_dev::IterStats>& stats, int* iterations, int* converged,
                    double* loop_ms) {
  const int64_t m = p.m;
  const int k = p.k;
  const double kd = static_cast<double>(k);
  double theta = cfg.has_theta0 ? cfg.theta0 : 1e-2 * pm_absmax * kd;
  if (theta <= 0) theta = 1e-2;
  theta = std::min(theta, cfg.theta_max);
  double res_scale = std::sqrt(kd) * std::sqrt(pm_norm2);
  if (res_scale == 0) res_scale = 1.0;
  const double mean = pm_sum / static_cast<double>(std::max<int64_t>(observed, 1));

  CnnmHandles hd;
  const size_t mk = static_cast<size_t>(m) * k;
  DBuf<double> dpm(m), dK(static_cast<size_t>(k) * k), Y(mk), Wa(mk), Z(mk), TMP(mk), n2(k);
  icnnm_dev::CGeo g{static_cast<int>(p.dims[0]), static_cast<int>(p.dims[1]),
                    static_cast<int>(p.dims[2]), static_cast<int>(p.kd[0]),
                    static_cast<int>(p.kd[1]), static_cast<int>(p.kd[2]), m, k};
  const int gx_up = static_cast<int>(std::min<int64_t>((m + 255) / 256, 592));
  const int gx_col = static_cast<int>(std::min<int64_t>((m + 255) / 256, 64));
  const int gx_el = grid_for(static_cast<int64_t>(mk), 256);
  DBuf<double> part_up(static_cast<size_t>(gx_up) * 3), part_gap(static_cast<size_t>(gx_col) * k),
      part_zn(static_cast<size_t>(gx_col) * k), red(2 * static_cast<size_t>(k));
  std::vector<double> hup(static_cast<size_t>(gx_up) * 3), hred(2 * static_cast<size_t>(k));
  CK(cudaMemcpyAsync(dK.p, K_colmajor, dK.bytes(), cudaMemcpyHostToDevice, hd.s));
  CK(cudaMemsetAsync(Y.p, 0, Y.bytes(), hd.s));
  icnnm_dev::f64_init<<<grid_for(m, 256), 256, 0, hd.s>>>(m, dM, dmask,
                                                          cfg.init_fill == ICNNM_INIT_MEAN, mean,
                                                          dpm.p, dL);
  CKL();
  const double one = 1.0, zero = 0.0;
  const int mi = static_cast<int>(m);
  // AKL = A(L) K: im2col (never kept between iterations) + DGEMM; K(s, j) = K_colmajor[j k + s]
  auto forward = [&]() {
    icnnm_dev::cnnm_prep<<<dim3(gx_col, k), 256, 0, hd.s>>>(g, dL, nullptr, 0.0, TMP.p);
    CKL();
    CKB(cublasDgemm(hd.b, CUBLAS_OP_N, CUBLAS_OP_N, mi, k, k, &one, TMP.p, mi, dK.p, k, &zero,
                    Wa.p, mi));
  };
  forward();  // Y = 0: Wa = AKL
  stats.assign(static_cast<size_t>(std::max(cfg.max_iters, 1)), icnnm_dev::IterStats{});
  *iterations = 0;
  *converged = 0;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, hd.s));
  for (int it = 0; it < cfg.max_iters; ++it) {
    const double tau = 1.0 / theta;
    // Z = prox_l21(Wa, 1/theta)                                 (solver.cpp:108, :42-50)
    CK(cudaMemsetAsync(n2.p, 0, n2.bytes(), hd.s));
    icnnm_dev::icnnm_colnorm2<<<k, 256, 0, hd.s>>>(m, k, Wa.p, n2.p);
    icnnm_dev::icnnm_colscale<<<gx_el, 256, 0, hd.s>>>(m, k, Wa.p, n2.p, tau, Z.p);
    // WK = (Y + theta Z) K^T -> the Wa buffer (Wa is rebuilt below)   (:110)
    icnnm_dev::f64_ypz<<<gx_el, 256, 0, hd.s>>>(static_cast<int64_t>(mk), Y.p, Z.p, theta, TMP.p);
    CKL();
    CKB(cublasDgemm(hd.b, CUBLAS_OP_N, CUBLAS_OP_T, mi, k, k, &one, TMP.p, mi, dK.p, k, &zero,
                    Wa.p, mi));
    // adjoint gather + L update                                  (:111-120)
    icnnm_dev::f64_update<<<gx_up, 256, 0, hd.s>>>(g, Wa.p, theta, cfg.lambda, dpm.p, dmask, dL,
                                                    part_up.p);
    CKL();
    forward();                                                   // :121
    const double theta_next = std::min(theta * cfg.theta_growth, cfg.theta_max);
    icnnm_dev::f64_dual<<<dim3(gx_col, k), 256, 0, hd.s>>>(m, k, Z.p, Y.p, theta,
                                                           1.0 / theta_next, Wa.p, part_gap.p,
                                                           part_zn.p);
    CKL();
    CK(cudaMemsetAsync(red.p, 0, red.bytes(), hd.s));
    icnnm_dev::icnnm_gram_reduce<<<grid_for(k, 256), 256, 0, hd.s>>>(k, gx_col, part_gap.p,
                                                                     red.p);
    icnnm_dev::icnnm_gram_reduce<<<grid_for(k, 256), 256, 0, hd.s>>>(k, gx_col, part_zn.p,
                                                                     red.p + k);
    CKL();
    CK(cudaMemcpyAsync(hup.data(), part_up.p, part_up.bytes(), cudaMemcpyDeviceToHost, hd.s));
    CK(cudaMemcpyAsync(hred.data(), red.p, red.bytes(), cudaMemcpyDeviceToHost, hd.s));
    CK(cudaStreamSynchronize(hd.s));
    icnnm_dev::IterStats& q = stats[it];
    for (int b = 0; b < gx_up; ++b) {
      q.dl2 += hup[3 * b];
      q.l2o += hup[3 * b + 1];
      q.fit += hup[3 * b + 2];
    }
    for (int c = 0; c < k; ++c) {
      q.gap2 += hred[c];
      q.z2 += hred[k + c];
      q.l21 += std::sqrt(hred[k + c]);
    }
    const double l_change = std::sqrt(q.dl2) / std::max(std::sqrt(q.l2o), 1e-300);
    const double residual = std::sqrt(q.gap2) / res_scale;
    theta = theta_next;
    *iterations = it + 1;
    if (residual < cfg.tol_primal || l_change < cfg.tol_change) {  // :136-139
      *converged = 1;
      break;
    }
  }
  CK(cudaEventRecord(e1, hd.s));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *loop_ms = ms;
}

}  // namespace icnnm_host

using namespace icnnm_host;

extern "C" int icnnm_cuda_cnnm_solve(int order, const int64_t* dims, const double* M_obs,
                                     const double* mask, const int64_t* kdims,
                                     const icnnm_solver_config* cfg, int device, double* L_out,
                                     icnnm_solve_report* report) {
  return guard([&] {
    validate_cfg(cfg);                                  // solver.cpp:66
    Problem p = make_problem(order, dims, kdims);       // :67
    if (!M_obs || !mask || !L_out || !report) invalid("solve: null input");
    DeviceScope ds(device);
    cnnm_solve_impl(p, M_obs, mask, *cfg, L_out, report);
  });
}
