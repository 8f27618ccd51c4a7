// Symmetric eigendecomposition for the PCA rotation (Theorem 1: the principal
// directions are the stationary points Sigma w = lambda w). fp64, host side (D x D, build time):
// Householder reduction to tridiagonal form, then implicit symmetric QR steps with Wilkinson
// shifts and Givens bulge chasing (Golub & Van Loan, Alg. 8.3.1 / 8.3.2), eigenvectors accumulated.
#include <cmath>
#include <vector>

#include "dade_internal.h"

namespace dade {

void sym_eig(int n, const double* Ain, double* eigval, double* Qcm /* column-major n x n */) {
  std::vector<double> A(Ain, Ain + (size_t)n * n);  // row-major, symmetric
  std::vector<double> Q((size_t)n * n, 0.0);        // row-major accumulation
  for (int i = 0; i < n; ++i) Q[(size_t)i * n + i] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[(size_t)i * n + j]; };
  auto q = [&](int i, int j) -> double& { return Q[(size_t)i * n + j]; };
  std::vector<double> v(n), p(n), w(n);
  // ---- Householder tridiagonalisation
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;  // length of x = A[k+1.., k]
    double xn2 = 0.0;
    for (int i = 0; i < m; ++i) { v[i] = a(k + 1 + i, k); xn2 += v[i] * v[i]; }
    const double xn = std::sqrt(xn2);
    if (xn == 0.0) continue;
    const double alpha = v[0] > 0 ? -xn : xn;
    v[0] -= alpha;
    double vtv = 0.0;
    for (int i = 0; i < m; ++i) vtv += v[i] * v[i];
    if (vtv == 0.0) continue;
    const double beta = 2.0 / vtv;
    // p = beta * A22 v
    for (int i = 0; i < m; ++i) {
      const double* row = &A[(size_t)(k + 1 + i) * n + (k + 1)];
      double s = 0.0;
      for (int j = 0; j < m; ++j) s += row[j] * v[j];
      p[i] = beta * s;
    }
    double ptv = 0.0;
    for (int i = 0; i < m; ++i) ptv += p[i] * v[i];
    const double K = 0.5 * beta * ptv;
    for (int i = 0; i < m; ++i) w[i] = p[i] - K * v[i];
    for (int i = 0; i < m; ++i) {
      double* row = &A[(size_t)(k + 1 + i) * n + (k + 1)];
      const double vi = v[i], wi = w[i];
      for (int j = 0; j < m; ++j) row[j] -= vi * w[j] + wi * v[j];
    }
    a(k + 1, k) = alpha;
    a(k, k + 1) = alpha;
    for (int i = 1; i < m; ++i) { a(k + 1 + i, k) = 0.0; a(k, k + 1 + i) = 0.0; }
    // Q[:, k+1:] -= beta * (Q[:, k+1:] v) v^T
    for (int r = 0; r < n; ++r) {
      double* row = &Q[(size_t)r * n + (k + 1)];
      double s = 0.0;
      for (int j = 0; j < m; ++j) s += row[j] * v[j];
      s *= beta;
      for (int j = 0; j < m; ++j) row[j] -= s * v[j];
    }
  }
  std::vector<double> d(n), e(n > 0 ? n : 1, 0.0);
  for (int i = 0; i < n; ++i) d[i] = a(i, i);
  for (int i = 0; i + 1 < n; ++i) e[i] = a(i + 1, i);
  // ---- implicit symmetric tridiagonal QR with Wilkinson shift
  const double eps = 2.220446049250313e-16;
  int hi = n - 1;
  int iter = 0;
  while (hi > 0) {
    if (std::fabs(e[hi - 1]) <= eps * (std::fabs(d[hi - 1]) + std::fabs(d[hi]))) {
      e[hi - 1] = 0.0;
      --hi;
      iter = 0;
      continue;
    }
    int lo = hi - 1;
    while (lo > 0 && std::fabs(e[lo - 1]) > eps * (std::fabs(d[lo - 1]) + std::fabs(d[lo]))) --lo;
    if (++iter > 60 * n) throw Error(DADE_ERR_CUDA, "eigensolver did not converge");
    const double dl = 0.5 * (d[hi - 1] - d[hi]);
    const double b2 = e[hi - 1] * e[hi - 1];
    const double sg = dl >= 0 ? 1.0 : -1.0;
    const double mu = d[hi] - b2 / (dl + sg * std::sqrt(dl * dl + b2));
    double x = d[lo] - mu, z = e[lo];
    for (int k = lo; k < hi; ++k) {
      const double r = std::hypot(x, z);
      const double c = r == 0.0 ? 1.0 : x / r, s = r == 0.0 ? 0.0 : z / r;
      if (k > lo) e[k - 1] = r;
      const double app = d[k], aqq = d[k + 1], apq = e[k];
      d[k] = c * c * app + 2.0 * c * s * apq + s * s * aqq;
      d[k + 1] = s * s * app - 2.0 * c * s * apq + c * c * aqq;
      e[k] = c * s * (aqq - app) + (c * c - s * s) * apq;
      if (k + 1 < hi) {
        z = s * e[k + 1];
        e[k + 1] = c * e[k + 1];
        x = e[k];
      }
      for (int r2 = 0; r2 < n; ++r2) {
        const double qp = q(r2, k), qq = q(r2, k + 1);
        q(r2, k) = c * qp + s * qq;
        q(r2, k + 1) = -s * qp + c * qq;
      }
    }
  }
  for (int i = 0; i < n; ++i) eigval[i] = d[i];
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) Qcm[(size_t)c * n + r] = q(r, c);
}

}  // namespace dade
