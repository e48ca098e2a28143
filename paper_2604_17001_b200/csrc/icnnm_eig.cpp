// Host symmetric eigensolver for the basis-learning stage (north-star (e):
// "the small k x k eigensolve stays on host").  Replaces Eigen's
// SelfAdjointEigenSolver used by psd_eig_sorted
// (/root/reference/proj/core/src/spectral.cpp:87-98).
//
// Algorithm: Householder reduction to symmetric tridiagonal form with the
// orthogonal transform accumulated, then the implicit-shift QL iteration on
// the tridiagonal matrix (the EISPACK tred2/tql2 pair, restated).  The
// transform is kept transposed during QL so every Givens rotation touches two
// contiguous rows.  Output: eigenvalues in DESCENDING order with eigenvectors
// as columns (column-major), matching the reversed order of spectral.cpp:93-95.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

namespace {

// Householder tridiagonalisation. V (row-major n x n) holds A on entry and the
// accumulated orthogonal transform on exit; d = diagonal, e = sub-diagonal
// (e[0] unused).
void householder_tridiag(int n, std::vector<double>& V, std::vector<double>& d,
                         std::vector<double>& e) {
  auto at = [&](int r, int c) -> double& { return V[static_cast<size_t>(r) * n + c]; };
  for (int j = 0; j < n; ++j) d[j] = at(n - 1, j);
  for (int i = n - 1; i > 0; --i) {
    double scale = 0.0, h = 0.0;
    for (int q = 0; q < i; ++q) scale += std::fabs(d[q]);
    if (scale == 0.0) {
      e[i] = d[i - 1];
      for (int j = 0; j < i; ++j) {
        d[j] = at(i - 1, j);
        at(i, j) = 0.0;
        at(j, i) = 0.0;
      }
    } else {
      for (int q = 0; q < i; ++q) {
        d[q] /= scale;
        h += d[q] * d[q];
      }
      double f = d[i - 1];
      double g = std::sqrt(h);
      if (f > 0) g = -g;
      e[i] = scale * g;
      h -= f * g;
      d[i - 1] = f - g;
      for (int j = 0; j < i; ++j) e[j] = 0.0;
      // e = A u (lower triangle of the active block is stored in V)
      for (int j = 0; j < i; ++j) {
        f = d[j];
        at(j, i) = f;
        g = e[j] + at(j, j) * f;
        for (int q = j + 1; q <= i - 1; ++q) {
          g += at(q, j) * d[q];
          e[q] += at(q, j) * f;
        }
        e[j] = g;
      }
      f = 0.0;
      for (int j = 0; j < i; ++j) {
        e[j] /= h;
        f += e[j] * d[j];
      }
      const double hh = f / (h + h);
      for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
      for (int j = 0; j < i; ++j) {
        f = d[j];
        g = e[j];
        for (int q = j; q <= i - 1; ++q) at(q, j) -= (f * e[q] + g * d[q]);
        d[j] = at(i - 1, j);
        at(i, j) = 0.0;
      }
    }
    d[i] = h;
  }
  // Accumulate the Householder reflections.
  for (int i = 0; i < n - 1; ++i) {
    at(n - 1, i) = at(i, i);
    at(i, i) = 1.0;
    const double h = d[i + 1];
    if (h != 0.0) {
      for (int q = 0; q <= i; ++q) d[q] = at(q, i + 1) / h;
      for (int j = 0; j <= i; ++j) {
        double g = 0.0;
        for (int q = 0; q <= i; ++q) g += at(q, i + 1) * at(q, j);
        for (int q = 0; q <= i; ++q) at(q, j) -= g * d[q];
      }
    }
    for (int q = 0; q <= i; ++q) at(q, i + 1) = 0.0;
  }
  for (int j = 0; j < n; ++j) {
    d[j] = at(n - 1, j);
    at(n - 1, j) = 0.0;
  }
  at(n - 1, n - 1) = 1.0;
  e[0] = 0.0;
}

// Implicit QL on the tridiagonal (d, e); Vt (row-major) holds the transform
// TRANSPOSED: row i of Vt is column i of V.  Returns false if not converged.
bool tridiag_ql(int n, std::vector<double>& Vt, std::vector<double>& d, std::vector<double>& e) {
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = std::ldexp(1.0, -52);
  for (int l = 0; l < n; ++l) {
    tst1 = std::max(tst1, std::fabs(d[l]) + std::fabs(e[l]));
    int m = l;
    while (m < n) {
      if (std::fabs(e[m]) <= eps * tst1) break;
      ++m;
    }
    if (m == n) m = n - 1;
    if (m > l) {
      int iter = 0;
      do {
        if (++iter > 200) return false;
        double g = d[l];
        double p = (d[l + 1] - g) / (2.0 * e[l]);
        double r = std::hypot(p, 1.0);
        if (p < 0) r = -r;
        d[l] = e[l] / (p + r);
        d[l + 1] = e[l] * (p + r);
        const double dl1 = d[l + 1];
        double h = g - d[l];
        for (int i = l + 2; i < n; ++i) d[i] -= h;
        f += h;
        p = d[m];
        double c = 1.0, c2 = c, c3 = c;
        const double el1 = e[l + 1];
        double s = 0.0, s2 = 0.0;
        for (int i = m - 1; i >= l; --i) {
          c3 = c2;
          c2 = c;
          s2 = s;
          g = c * e[i];
          h = c * p;
          r = std::hypot(p, e[i]);
          e[i + 1] = s * r;
          s = e[i] / r;
          c = p / r;
          p = c * d[i] - s * g;
          d[i + 1] = h + s * (c * g + s * d[i]);
          double* vi = Vt.data() + static_cast<size_t>(i) * n;
          double* vi1 = Vt.data() + static_cast<size_t>(i + 1) * n;
          for (int q = 0; q < n; ++q) {
            const double hv = vi1[q];
            vi1[q] = s * vi[q] + c * hv;
            vi[q] = c * vi[q] - s * hv;
          }
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = c * p;
      } while (std::fabs(e[l]) > eps * tst1);
    }
    d[l] += f;
    e[l] = 0.0;
  }
  return true;
}

}  // namespace

extern "C" int icnnm_host_symeig_impl(int n, const double* G, double* evals_desc,
                                      double* evecs) {
  if (n == 1) {
    evals_desc[0] = G[0];
    evecs[0] = 1.0;
    return 0;
  }
  std::vector<double> V(static_cast<size_t>(n) * n), d(n), e(n);
  // G is symmetric; column-major == row-major.
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) V[static_cast<size_t>(r) * n + c] = G[static_cast<size_t>(c) * n + r];
  householder_tridiag(n, V, d, e);
  std::vector<double> Vt(static_cast<size_t>(n) * n);
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) Vt[static_cast<size_t>(c) * n + r] = V[static_cast<size_t>(r) * n + c];
  V.clear();
  V.shrink_to_fit();
  if (!tridiag_ql(n, Vt, d, e)) return 1;
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] > d[b]; });
  for (int i = 0; i < n; ++i) {
    evals_desc[i] = d[idx[i]];
    const double* src = Vt.data() + static_cast<size_t>(idx[i]) * n;
    std::copy(src, src + n, evecs + static_cast<size_t>(i) * n);
  }
  return 0;
}
