// Native 1-D bases in long double (see wk_basis.h).
#include "wk_basis.h"

#include <cmath>
#include <stdexcept>

namespace wk {

namespace {
// Legendre P_n and P_n' on [-1,1] by the three-term recurrence.
void legendre(int n, long double x, long double& p, long double& dp) {
  long double p0 = 1.0L, p1 = x;
  if (n == 0) { p = 1.0L; dp = 0.0L; return; }
  for (int k = 2; k <= n; ++k) {
    long double pk = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1; p1 = pk;
  }
  p = p1;
  // P_n' = n (x P_n - P_{n-1}) / (x^2 - 1); endpoints handled by callers
  dp = n * (x * p1 - p0) / (x * x - 1.0L);
}
const long double kPi = 3.141592653589793238462643383279502884L;
}  // namespace

void gauss_rule(int n, std::vector<long double>& x, std::vector<long double>& w) {
  if (n < 1) throw std::invalid_argument("gauss_rule needs n >= 1");
  x.assign(n, 0.0L); w.assign(n, 0.0L);
  for (int i = 0; i < n; ++i) {
    long double t = std::cos(kPi * (i + 0.75L) / (n + 0.5L));
    for (int it = 0; it < 100; ++it) {
      long double p, dp;
      legendre(n, t, p, dp);
      long double dt = p / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-19L) break;
    }
    long double p, dp;
    legendre(n, t, p, dp);
    // descending t -> ascending points on [0,1]
    x[n - 1 - i] = 0.5L * (t + 1.0L);
    w[n - 1 - i] = 1.0L / ((1.0L - t * t) * dp * dp);  // 2/(..) halved
  }
}

void gauss_lobatto_rule(int n, std::vector<long double>& x, std::vector<long double>& w) {
  if (n < 2) throw std::invalid_argument("gauss_lobatto_rule needs n >= 2");
  x.assign(n, 0.0L); w.assign(n, 0.0L);
  const int m = n - 1;  // interior points are the roots of P_m'
  std::vector<long double> t(n);
  t[0] = -1.0L; t[m] = 1.0L;
  for (int i = 1; i < m; ++i) {
    long double s = -std::cos(kPi * i / m);
    for (int it = 0; it < 100; ++it) {
      // f = P_m', f' = (2 s P_m' - m(m+1) P_m) / (1 - s^2)
      long double p, dp;
      legendre(m, s, p, dp);
      long double d2 = (2.0L * s * dp - m * (m + 1) * p) / (1.0L - s * s);
      long double ds = dp / d2;
      s -= ds;
      if (std::fabs(ds) < 1e-19L) break;
    }
    t[i] = s;
  }
  for (int i = 0; i < n; ++i) {
    long double p, dp;
    legendre(m, t[i], p, dp);
    x[i] = 0.5L * (t[i] + 1.0L);
    w[i] = 1.0L / (n * (n - 1) * p * p);
  }
  x[0] = 0.0L; x[m] = 1.0L;
}

Mat lagrange(const std::vector<long double>& nodes, const std::vector<long double>& pts,
             bool deriv) {
  const int nn = (int)nodes.size(), np = (int)pts.size();
  Mat out((size_t)np * nn, 0.0L);
  for (int j = 0; j < nn; ++j) {
    long double denom = 1.0L;
    for (int q = 0; q < nn; ++q)
      if (q != j) denom *= nodes[j] - nodes[q];
    for (int i = 0; i < np; ++i) {
      long double xv = pts[i];
      if (!deriv) {
        long double num = 1.0L;
        for (int q = 0; q < nn; ++q)
          if (q != j) num *= xv - nodes[q];
        out[(size_t)i * nn + j] = num / denom;
      } else {
        long double acc = 0.0L;
        for (int r = 0; r < nn; ++r) {
          if (r == j) continue;
          long double prod = 1.0L;
          for (int q = 0; q < nn; ++q)
            if (q != j && q != r) prod *= xv - nodes[q];
          acc += prod;
        }
        out[(size_t)i * nn + j] = acc / denom;
      }
    }
  }
  return out;
}

Mat matmul(const Mat& a, const Mat& b, int m, int k, int n) {
  Mat c((size_t)m * n, 0.0L);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      long double s = 0.0L;
      for (int q = 0; q < k; ++q) s += a[(size_t)i * k + q] * b[(size_t)q * n + j];
      c[(size_t)i * n + j] = s;
    }
  return c;
}

Mat transpose(const Mat& a, int m, int n) {
  Mat t((size_t)m * n);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) t[(size_t)j * m + i] = a[(size_t)i * n + j];
  return t;
}

Mat inverse(const Mat& a_in, int n) {
  Mat a = a_in, inv((size_t)n * n, 0.0L);
  for (int i = 0; i < n; ++i) inv[(size_t)i * n + i] = 1.0L;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[(size_t)r * n + c]) > std::fabs(a[(size_t)piv * n + c])) piv = r;
    if (a[(size_t)piv * n + c] == 0.0L) throw std::runtime_error("singular matrix");
    if (piv != c)
      for (int j = 0; j < n; ++j) {
        std::swap(a[(size_t)c * n + j], a[(size_t)piv * n + j]);
        std::swap(inv[(size_t)c * n + j], inv[(size_t)piv * n + j]);
      }
    long double d = a[(size_t)c * n + c];
    for (int j = 0; j < n; ++j) { a[(size_t)c * n + j] /= d; inv[(size_t)c * n + j] /= d; }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      long double f = a[(size_t)r * n + c];
      if (f == 0.0L) continue;
      for (int j = 0; j < n; ++j) {
        a[(size_t)r * n + j] -= f * a[(size_t)c * n + j];
        inv[(size_t)r * n + j] -= f * inv[(size_t)c * n + j];
      }
    }
  }
  return inv;
}

std::vector<long double> g_nodes(int k) {
  std::vector<long double> x, w;
  gauss_rule(k + 1, x, w);
  return x;
}

std::vector<long double> gl_nodes(int k) {
  if (k == 0) return g_nodes(0);
  std::vector<long double> x, w;
  gauss_lobatto_rule(k + 1, x, w);
  return x;
}

Mat resize_gauss(int k_from, int k_to) {
  std::vector<long double> g_from, w_from, g_to, w_to;
  gauss_rule(k_from + 1, g_from, w_from);
  gauss_rule(k_to + 1, g_to, w_to);
  if (k_to >= k_from) return lagrange(g_from, g_to, false);
  // P = W_to^{-1} A_to^T W_mix A_from, mixed rule = (k_from+1)-point Gauss
  Mat a_to = lagrange(g_to, g_from, false);      // (n_from x n_to): L^to_j(x_mix_i)
  const int nf = k_from + 1, nt = k_to + 1;
  Mat p((size_t)nt * nf, 0.0L);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nf; ++j)
      p[(size_t)i * nf + j] = a_to[(size_t)j * nt + i] * w_from[j] / w_to[i];
  // a_from at its own points is the identity, so the product collapses
  return p;
}

}  // namespace wk
