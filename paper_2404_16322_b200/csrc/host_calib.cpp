// Host-side (fp64) parts of calibration (a3): the per-step logistic fit and the counter hash.
// Logistic regression with cross-entropy loss on features (dis', tau), reduced to
// sign(m1 * dis' + beta > tau). Reading R3: the BCE minimiser via damped Newton
// (IRLS) on standardised features with a 1e-8 ridge on the non-intercept weights.
#include <cmath>
#include <vector>

#include "dade_internal.h"

namespace dade {

uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static bool solve3(double H[3][3], const double g[3], double x[3]) {
  double M[3][4];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) M[i][j] = H[i][j];
    M[i][3] = g[i];
  }
  for (int c = 0; c < 3; ++c) {
    int piv = c;
    for (int r = c + 1; r < 3; ++r)
      if (std::fabs(M[r][c]) > std::fabs(M[piv][c])) piv = r;
    if (M[piv][c] == 0.0) return false;
    if (piv != c)
      for (int j = 0; j < 4; ++j) std::swap(M[c][j], M[piv][j]);
    for (int r = 0; r < 3; ++r) {
      if (r == c) continue;
      const double f = M[r][c] / M[c][c];
      for (int j = c; j < 4; ++j) M[r][j] -= f * M[c][j];
    }
  }
  for (int i = 0; i < 3; ++i) x[i] = M[i][3] / M[i][i];
  return true;
}

static inline double log1pexp(double z) {  // log(1 + e^z), overflow-free
  return z > 0 ? z + std::log1p(std::exp(-z)) : std::log1p(std::exp(z));
}

bool logistic_irls(const std::vector<double>& P, const std::vector<double>& tau,
                   const std::vector<double>& y, double ridge, int max_iter, double tol,
                   double* m1_out, double* beta_out) {
  const size_t n = P.size();
  double mP = 0, mt = 0;
  for (size_t i = 0; i < n; ++i) { mP += P[i]; mt += tau[i]; }
  mP /= (double)n;
  mt /= (double)n;
  double sP = 0, st = 0;
  for (size_t i = 0; i < n; ++i) {
    sP += (P[i] - mP) * (P[i] - mP);
    st += (tau[i] - mt) * (tau[i] - mt);
  }
  sP = std::sqrt(sP / (double)n);
  st = std::sqrt(st / (double)n);
  if (!(sP > 0)) sP = 1.0;
  if (!(st > 0)) st = 1.0;
  std::vector<double> f1(n), f2(n);
  for (size_t i = 0; i < n; ++i) { f1[i] = (P[i] - mP) / sP; f2[i] = (tau[i] - mt) / st; }
  const double reg[3] = {0.0, ridge, ridge};
  auto loss = [&](const double w[3]) {
    double L = 0;
    for (size_t i = 0; i < n; ++i) {
      const double z = w[0] + w[1] * f1[i] + w[2] * f2[i];
      L += log1pexp(z) - y[i] * z;
    }
    for (int j = 0; j < 3; ++j) L += 0.5 * reg[j] * w[j] * w[j];
    return L;
  };
  double w[3] = {0, 0, 0};
  double cur = loss(w);
  for (int it = 0; it < max_iter; ++it) {
    double g[3] = {0, 0, 0}, H[3][3] = {{0}};
    for (size_t i = 0; i < n; ++i) {
      const double z = w[0] + w[1] * f1[i] + w[2] * f2[i];
      const double p = 0.5 * (1.0 + std::tanh(0.5 * z));
      const double a[3] = {1.0, f1[i], f2[i]};
      const double r = y[i] - p, ww = p * (1.0 - p);
      for (int j = 0; j < 3; ++j) {
        g[j] += a[j] * r;
        for (int k = 0; k < 3; ++k) H[j][k] += a[j] * a[k] * ww;
      }
    }
    for (int j = 0; j < 3; ++j) { g[j] -= reg[j] * w[j]; H[j][j] += reg[j]; }
    double step[3];
    if (!solve3(H, g, step)) break;
    double t = 1.0, nw[3], nl = cur;
    for (int h = 0; h < 30; ++h) {
      for (int j = 0; j < 3; ++j) nw[j] = w[j] + t * step[j];
      nl = loss(nw);
      if (nl <= cur) break;
      t *= 0.5;
    }
    double mx = 0;
    for (int j = 0; j < 3; ++j) { w[j] = nw[j]; mx = std::fmax(mx, std::fabs(t * step[j])); }
    cur = nl;
    if (mx < tol) break;
  }
  const double wP = w[1] / sP, wt = w[2] / st;
  const double b = w[0] - w[1] * mP / sP - w[2] * mt / st;
  if (!(wt < 0) || !std::isfinite(wP) || !std::isfinite(wt)) { *m1_out = 1.0; *beta_out = 0.0; return false; }
  const double m1 = -wP / wt;
  if (!(m1 > 0) || !std::isfinite(m1)) { *m1_out = 1.0; *beta_out = 0.0; return false; }
  *m1_out = m1;
  *beta_out = -b / wt;
  return true;
}

// Several features (BSA-q: the ADC distance and the distance to the quantized
// centroid) — the same damped Newton / IRLS on standardised features (R3), k features + tau.
// F: n x k row-major. Returns the model m . f + beta > tau (m_i = -w_i / w_tau); flag (R29):
// w_tau >= 0, a non-finite weight or m_0 <= 0 -> m = e_0, beta = 0, false.
static bool solve_n(std::vector<double>& M, int n, std::vector<double>& x) {  // M: n x (n+1)
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(M[(size_t)r * (n + 1) + c]) > std::fabs(M[(size_t)piv * (n + 1) + c])) piv = r;
    if (M[(size_t)piv * (n + 1) + c] == 0.0) return false;
    if (piv != c)
      for (int j = 0; j <= n; ++j) std::swap(M[(size_t)c * (n + 1) + j], M[(size_t)piv * (n + 1) + j]);
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = M[(size_t)r * (n + 1) + c] / M[(size_t)c * (n + 1) + c];
      for (int j = c; j <= n; ++j) M[(size_t)r * (n + 1) + j] -= f * M[(size_t)c * (n + 1) + j];
    }
  }
  x.resize(n);
  for (int i = 0; i < n; ++i) x[i] = M[(size_t)i * (n + 1) + n] / M[(size_t)i * (n + 1) + i];
  return true;
}

bool logistic_irls_multi(const std::vector<double>& F, int k, const std::vector<double>& tau,
                         const std::vector<double>& y, double ridge, int max_iter, double tol,
                         std::vector<double>& m_out, double* beta_out) {
  const size_t n = tau.size();
  const int nw = k + 2;  // intercept, k features, tau
  std::vector<double> mean(k + 1, 0.0), sd(k + 1, 0.0);
  for (size_t i = 0; i < n; ++i) {
    for (int j = 0; j < k; ++j) mean[j] += F[i * k + j];
    mean[k] += tau[i];
  }
  for (auto& v : mean) v /= (double)n;
  for (size_t i = 0; i < n; ++i) {
    for (int j = 0; j < k; ++j) sd[j] += (F[i * k + j] - mean[j]) * (F[i * k + j] - mean[j]);
    sd[k] += (tau[i] - mean[k]) * (tau[i] - mean[k]);
  }
  for (auto& v : sd) { v = std::sqrt(v / (double)n); if (!(v > 0)) v = 1.0; }
  std::vector<double> A(n * nw);
  for (size_t i = 0; i < n; ++i) {
    A[i * nw] = 1.0;
    for (int j = 0; j < k; ++j) A[i * nw + 1 + j] = (F[i * k + j] - mean[j]) / sd[j];
    A[i * nw + 1 + k] = (tau[i] - mean[k]) / sd[k];
  }
  std::vector<double> reg(nw, ridge);
  reg[0] = 0.0;
  auto loss = [&](const std::vector<double>& w) {
    double L = 0;
    for (size_t i = 0; i < n; ++i) {
      double z = 0;
      for (int j = 0; j < nw; ++j) z += A[i * nw + j] * w[j];
      L += log1pexp(z) - y[i] * z;
    }
    for (int j = 0; j < nw; ++j) L += 0.5 * reg[j] * w[j] * w[j];
    return L;
  };
  std::vector<double> w(nw, 0.0), nwv(nw), step;
  double cur = loss(w);
  std::vector<double> M((size_t)nw * (nw + 1));
  for (int it = 0; it < max_iter; ++it) {
    std::fill(M.begin(), M.end(), 0.0);
    for (size_t i = 0; i < n; ++i) {
      double z = 0;
      for (int j = 0; j < nw; ++j) z += A[i * nw + j] * w[j];
      const double p = 0.5 * (1.0 + std::tanh(0.5 * z));
      const double r = y[i] - p, ww = p * (1.0 - p);
      for (int a = 0; a < nw; ++a) {
        M[(size_t)a * (nw + 1) + nw] += A[i * nw + a] * r;
        for (int b = 0; b < nw; ++b) M[(size_t)a * (nw + 1) + b] += A[i * nw + a] * A[i * nw + b] * ww;
      }
    }
    for (int j = 0; j < nw; ++j) {
      M[(size_t)j * (nw + 1) + nw] -= reg[j] * w[j];
      M[(size_t)j * (nw + 1) + j] += reg[j];
    }
    if (!solve_n(M, nw, step)) break;
    double t = 1.0, nl = cur;
    for (int h = 0; h < 30; ++h) {
      for (int j = 0; j < nw; ++j) nwv[j] = w[j] + t * step[j];
      nl = loss(nwv);
      if (nl <= cur) break;
      t *= 0.5;
    }
    double mx = 0;
    for (int j = 0; j < nw; ++j) { w[j] = nwv[j]; mx = std::fmax(mx, std::fabs(t * step[j])); }
    cur = nl;
    if (mx < tol) break;
  }
  const double wt = w[1 + k] / sd[k];
  double b = w[0] - w[1 + k] * mean[k] / sd[k];
  std::vector<double> wf(k);
  bool finite = std::isfinite(wt);
  for (int j = 0; j < k; ++j) {
    wf[j] = w[1 + j] / sd[j];
    b -= w[1 + j] * mean[j] / sd[j];
    finite = finite && std::isfinite(wf[j]);
  }
  m_out.assign(k, 0.0);
  m_out[0] = 1.0;
  *beta_out = 0.0;
  if (!(wt < 0) || !finite) return false;
  std::vector<double> mv(k);
  for (int j = 0; j < k; ++j) mv[j] = -wf[j] / wt;
  if (!(mv[0] > 0)) return false;
  for (double v : mv)
    if (!std::isfinite(v)) return false;
  m_out = mv;
  *beta_out = -b / wt;
  return true;
}

}  // namespace dade
