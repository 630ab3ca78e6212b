// host_math.cpp -- host-side fp64 steps of the hot path:
//   * complete elliptic integral K and Jacobi sn/cn/dn by the arithmetic-geometric mean
//     (descending Landen) with the COMPLEMENTARY parameter passed exactly, so that the
//     ill-conditioned case m' = 1 - lambda_min/lambda_max -> 1 loses no digits;
//   * the Hale-Higham-Trefethen rule in real arithmetic (eq. quad_points_and_locations,
//     P:1443-1469, through the Jacobi imaginary transform sn(ix|k) = i sc(x|k'),
//     cn(ix|k) = nc(x|k'), dn(ix|k) = dc(x|k'); reading G10);
//   * extreme eigenvalues of the Lanczos tridiagonal T_J by Sturm-sequence bisection.
// Independent of oracle/ (which evaluates the complex formula with mpmath).
#include <cmath>
#include <cstdint>
#include <algorithm>
#include <limits>
#include <vector>

#include "host_math.h"

namespace ciqh {

// AGM iteration a_{n+1} = (a_n + b_n)/2, b_{n+1} = sqrt(a_n b_n), c_{n+1} = (a_n - b_n)/2 started
// from (1, sqrt(m1), sqrt(m)) -- Abramowitz & Stegun 17.6 / 16.4.
static int agm_sequence(double m, double m1, double* a, double* c, int max_n) {
  double an = 1.0, bn = std::sqrt(m1);
  a[0] = 1.0;
  c[0] = std::sqrt(m);
  int n = 0;
  while (n + 1 < max_n && std::fabs(c[n]) > 1e-17 * a[n]) {
    double a1 = 0.5 * (an + bn);
    double c1 = 0.5 * (an - bn);
    double b1 = std::sqrt(an * bn);
    an = a1;
    bn = b1;
    ++n;
    a[n] = an;
    c[n] = c1;
  }
  return n;
}

double ellipk_comp(double m, double m1) {
  // K(m) = pi / (2 AGM(1, sqrt(1 - m)))
  double a[64], c[64];
  int n = agm_sequence(m, m1, a, c, 64);
  return M_PI / (2.0 * a[n]);
}

void ellipj_comp(double u, double m, double m1, double* sn, double* cn, double* dn) {
  if (m == 0.0) {
    *sn = std::sin(u);
    *cn = std::cos(u);
    *dn = 1.0;
    return;
  }
  double a[64], c[64];
  int n = agm_sequence(m, m1, a, c, 64);
  double phi = std::ldexp(a[n] * u, n);  // 2^n a_n u
  double phi_prev = phi;
  for (int i = n; i >= 1; --i) {
    phi_prev = phi;
    phi = 0.5 * (phi + std::asin(c[i] / a[i] * std::sin(phi)));
  }
  *sn = std::sin(phi);
  *cn = std::cos(phi);
  *dn = (n >= 1) ? std::cos(phi) / std::cos(phi_prev - phi) : std::sqrt(1.0 - m * (*sn) * (*sn));
}

int hht_rule(double lambda_min, double lambda_max, int Q, double* t, double* w) {
  if (!(lambda_min > 0.0) || !(lambda_max > 0.0) || Q < 1) return -1;
  // kappa clamped to >= 1 + 1e-8 (k < 1).
  double lmax = std::fmax(lambda_max, lambda_min * (1.0 + 1e-8));
  double k2 = lambda_min / lmax;  // k^2, k = 1/sqrt(kappa)
  double mp = 1.0 - k2;           // parameter of k' (m' = k'^2)
  double kp = ellipk_comp(mp, k2);  // K'(k) = K(k')
  double scale = 2.0 * std::sqrt(lambda_min) * kp / (M_PI * Q);
  for (int q = 1; q <= Q; ++q) {
    double u = (q - 0.5) / Q;  // u_q
    double sn, cn, dn;
    ellipj_comp(u * kp, mp, k2, &sn, &cn, &dn);
    // sigma_q^2 = lambda_min sn(i u K'|k)^2 = -lambda_min sc(u K'|k')^2  -> t_q = lambda_min sc^2
    // w~_q = -(2 sqrt(lmin)/(pi Q)) K' cn(i.)dn(i.) = -(2 sqrt(lmin) K'/(pi Q)) dn/cn^2 -> w_q = -w~_q
    double sc = sn / cn;
    t[q - 1] = lambda_min * sc * sc;
    w[q - 1] = scale * dn / (cn * cn);
    if (!std::isfinite(t[q - 1]) || !std::isfinite(w[q - 1]) || !(t[q - 1] > 0) || !(w[q - 1] > 0))
      return -2;
  }
  return 0;
}

// Number of eigenvalues of the tridiagonal (alpha, beta) strictly less than x (Sturm count).
static int sturm_count(const double* alpha, const double* beta, int m, double x) {
  int count = 0;
  double d = 1.0;
  for (int i = 0; i < m; ++i) {
    double b2 = (i > 0) ? beta[i - 1] * beta[i - 1] : 0.0;
    d = alpha[i] - x - ((i > 0) ? b2 / d : 0.0);
    if (d == 0.0) d = -std::numeric_limits<double>::min() * 1e6;  // perturb off the pole
    if (d < 0.0) ++count;
  }
  return count;
}

int tridiag_extremes(const double* alpha, const double* beta, int m, double* emin, double* emax) {
  if (m < 1) return -1;
  double lo = std::numeric_limits<double>::infinity(), hi = -lo;
  for (int i = 0; i < m; ++i) {  // Gershgorin interval
    double r = 0.0;
    if (i > 0) r += std::fabs(beta[i - 1]);
    if (i < m - 1) r += std::fabs(beta[i]);
    lo = std::fmin(lo, alpha[i] - r);
    hi = std::fmax(hi, alpha[i] + r);
  }
  double span = std::fmax(hi - lo, std::fmax(std::fabs(lo), std::fabs(hi)) * 1e-300);
  // smallest eigenvalue: largest x with count(x) == 0
  double a = lo - 1e-12 * span, b = hi + 1e-12 * span;
  for (int it = 0; it < 200 && (b - a) > 4e-16 * std::fmax(std::fabs(a), std::fabs(b)); ++it) {
    double mid = 0.5 * (a + b);
    if (sturm_count(alpha, beta, m, mid) >= 1) b = mid; else a = mid;
  }
  *emin = 0.5 * (a + b);
  a = lo - 1e-12 * span;
  b = hi + 1e-12 * span;
  for (int it = 0; it < 200 && (b - a) > 4e-16 * std::fmax(std::fabs(a), std::fabs(b)); ++it) {
    double mid = 0.5 * (a + b);
    if (sturm_count(alpha, beta, m, mid) >= m) b = mid; else a = mid;
  }
  *emax = 0.5 * (a + b);
  return 0;
}

// Cyclic Jacobi eigendecomposition of a symmetric n x n matrix a (row-major, destroyed):
// eigenvalues -> w (descending), eigenvectors -> columns of v (row-major n x n).
int sym_eig_jacobi(double* a, int n, double* w, double* v) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) v[i * n + j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += a[i * n + j] * a[i * n + j];
        if (i != j) off += a[i * n + j] * a[i * n + j];
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double app = a[p * n + p], aqq = a[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // rotate columns p, q
          const double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - s * akq;
          a[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // rotate rows p, q
          const double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - s * aqk;
          a[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - s * vkq;
          v[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  // sort descending
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int x, int y) { return a[x * n + x] > a[y * n + y]; });
  std::vector<double> vs((size_t)n * n);
  for (int j = 0; j < n; ++j) {
    w[j] = a[idx[j] * n + idx[j]];
    for (int i = 0; i < n; ++i) vs[(size_t)i * n + j] = v[i * n + idx[j]];
  }
  std::copy(vs.begin(), vs.end(), v);
  return 0;
}

}  // namespace ciqh
