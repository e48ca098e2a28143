// Shared device-side declarations of the ICNNM hot-path kernels.
//
// Tensor geometry follows the reference's conventions
// (/root/reference/proj/core/include/icnnm/tensor.hpp:64-68, fft.cpp:78-90):
// row-major [H, W, T] (lower orders are padded with leading 1s), kernel taps
// corner-anchored and flattened row-major over the (kh, kw, kt) box
// (conv_op.cpp:42-44,94).  Forward:  T[i, j] = sum_s L[(i - s) mod dims] K[s, j].
// Adjoint: out[i] = sum_s U[(i + s) mod dims, s].
#pragma once
#include <cstdint>

namespace icnnm_dev {

// Programmatic dependent launch (PDL).  The hot-loop kernels launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start (prologue:
// TMEM alloc, barrier init, tap tables) while their predecessor finishes;
// pdl_wait() blocks until the predecessor grid has completed and its writes
// are visible, and every kernel of the chain executes it before its first
// dependent global access, so completion stays transitive.  Without the
// attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

constexpr int BM = 128;   // voxels per tile (one brick)
constexpr int BN = 64;    // output columns per N-tile
constexpr int BK = 32;    // reduction chunk

// Geometry of one launch.  The voxel tile is a brick (bh, bw, bt) with
// bh*bw*bt == 128 and bt a multiple of 8; bricks tile the (H, W, T) box
// (voxels outside the tensor are masked).  W rows are brick-ordered:
// row = brick*128 + local voxel, so a CTA's 128 rows are contiguous.
// Deterministic adjoint output (icnnm_tc.cu flush, icnnm_adj_q2f).  Every
// partial sum s a CTA flushes is split into two fp32 numbers on fixed grids,
//   hi = rint(s / qh) qh,   lo = rint((s - hi) / ql) ql,   ql = qh 2^-17,
// and added to the voxel's {hi, lo} pair with one vector reduction
// (red.global.add.v2.f32).  With |adj_i| <= sum over k taps of |U[v, s]| <=
// amax ||K[s, :]||_1 <= amax sqrt(k) k (K orthogonal, amax the coef kernel's
// bound on |W_vj c_j|) and qh = 2^eh >= 2 amax k sqrt(k) 2^-23, every running
// hi sum is a multiple of qh below 2^24 qh and every lo sum (<= 2^6
// contributions of at most qh/2) a multiple of ql below 2^24 ql: all fp32 adds
// are exact, so the result does not depend on the order in which CTAs flush.
// What is dropped is at most ql/2 = 2^-41 of the bound per contribution.
struct AdjGrid {
  float qh, inv_qh, ql, inv_ql;
};
__device__ __forceinline__ AdjGrid adj_grid(double amax, int k) {
  int ex = 0;
  if (amax > 0.0 && amax < 1e300)
    frexp(2.0 * amax * static_cast<double>(k) * sqrt(static_cast<double>(k)), &ex);
  int eh = ex - 23;
  eh = eh < -100 ? -100 : (eh > 100 ? 100 : eh);  // the lo grid stays above fp32 subnormals
  AdjGrid g;
  g.qh = ldexpf(1.f, eh);
  g.inv_qh = ldexpf(1.f, -eh);
  g.ql = ldexpf(1.f, eh - 17);
  g.inv_ql = ldexpf(1.f, 17 - eh);
  return g;
}

struct Geo {
  int H, W, T;          // voxels owned by this launch (H = slab rows)
  int kh, kw, kt;       // kernel box
  int bh, bw, bt;       // brick
  int nbh, nbw, nbt;    // bricks per axis
  int HH, HW, HT;       // halo box = brick + kernel - 1
  int k;                // taps
  int kp;               // W / K columns padded to a multiple of BN
  int ktp;              // taps padded to a multiple of BN
  int Hsrc;             // rows of the source (L~) / target (adj) buffer
  int hoff;             // buffer row = h + hoff   (h may be negative)
  int wrapH;            // 1: periodic in H over Hsrc rows; 0: slab buffer
  int vmap;             // tcgen05 engines: voxel order within a brick (TMEM lane / W row)
                        // 0: v = (vh*bw + vw)*bt + vt;  1: v = (vw*bh + vh)*bt + vt
};

// Per-iteration scalars, written by the coefficient kernel and read by the
// other kernels of the same iteration (stream order, no host round trip).
struct IterState {
  int it;          // current iteration
  int next_it;     // iteration the next coef launch will start
  int active;      // 0 once converged or max_iters reached
  int converged;
  int max_iters;
  int pad0;
  double theta;    // theta_it
  double r;        // theta_it / theta_{it+1}
  double adj_amax; // max_j min(n_j, 1/theta) >= |W_vj c_j|: F16x3 adjoint operand scale
};

// Per-iteration reductions (fp64).
struct IterStats {
  double l21;   // sum_j max(0, n_j - 1/theta)      = ||Z||_{2,1}
  double z2;    // sum_j (1-c_j)^2 n_j^2            = ||Z||_F^2
  double dl2;   // ||L_{t+1} - L_t||^2
  double l2o;   // ||L_t||^2
  double fit;   // ||mask (L_{t+1} - M)||^2
  double ip;    // <k L_t - V_t - adj_t, L_{t+1}>   (= <Z_t, A(L_{t+1})K>)
  double ln2;   // ||L_{t+1}||^2
  double gap2;  // exact ||Z_t - A(L_{t+1})K||^2 (exact_residual mode), else 0
};

// Deterministic-reduction buffers of one iteration (null: not used).
struct Partials {
  const double* npart;  // forward column partials [nrows][kp]
  int nrows;
  const double* upart;  // update report partials [urows][8]
  int urows;
  const double* gpart;  // exact-residual gap partials [grows]
  int grows;
};

}  // namespace icnnm_dev

// Kernel declarations (defined in icnnm_kernels.cu; launched from the host
// driver, which is a separate translation unit).
namespace icnnm_dev {
__global__ void icnnm_fwd_ffma(Geo g, const float* Lt, const float* Krm, float* Wm,
                               const float* cvec, const IterState* st, double* norm2,
                               int mode);
__global__ void icnnm_adj_ffma(Geo g, const float* Wm, const float* KT, const float* cvec,
                               float* adj, const IterState* st, int mode);
__global__ void icnnm_coef(IterState* st, const double* theta, double* red, float* cvec,
                           IterStats* stats, int k, int kp, double kd, double res_scale,
                           double tol_p, double tol_c, double floor_rel, int exact, Partials P);
__global__ void icnnm_fold(Partials P, int kp, double* red);
__global__ void icnnm_adj_q2f(int64_t n, const IterState* st, float2* adjq, float* adj);
constexpr int UPD_U = 4;  // elements in flight per thread (icnnm_update)
__global__ void icnnm_update(int64_t m, const IterState* st, double lambda, double kd,
                             float* adj, double* L, double* V, const float* pm,
                             const float* mask, float* Lt, double* slot, float* Lr,
                             double* upart, float2* adjq);
__global__ void icnnm_add_rows(int64_t n, float* dst, float* src);
__global__ void icnnm_setup(int64_t m, const double* M, const double* msk, int mean_fill,
                            double mean, float* pm, float* maskf, double* L, double* V,
                            float* Lt);
__global__ void icnnm_gram_lags(int H, int W, int T, int kh, int kw, int kt, int bh, int bw,
                                int bt, const double* X, double* R);
__global__ void icnnm_gram_reduce(int64_t n, int ny, const double* partial, double* R_out);
constexpr int GRAM_KT_MAX = 9;  // register-tiled Gram kernel: largest frame-kernel size
void* gram_lags_rt_ptr(int kt);  // icnnm_gram_lags_rt<kt>(H, W, T, kw, bh, bw, bt, X, R) or null
__global__ void icnnm_gram_reduce_sym(int kh, int nl, int ny, const double* partial,
                                      double* R_out);
__global__ void icnnm_dfma_probe(double* out, int iters, double seed);
__global__ void icnnm_colnorm2(int64_t rows, int64_t cols, const double* W, double* out);
__global__ void icnnm_colscale(int64_t rows, int64_t cols, const double* W, const double* n2,
                               double tau, double* Z);
__global__ void icnnm_f64_to_f32(int64_t n, const double* a, float* b);
__global__ void icnnm_ffma_probe(float* out, int iters, float seed);
constexpr int GRAM_LPT_HOST = 8;
}  // namespace icnnm_dev
