// host_stats.cpp -- host-side critical values and radius schedule.
//
// The F critical value F_c(t) = quantile(1 - alpha_F; n - 1, n (t J - 1))
// depends only on the held-iteration count t, so the context tabulates it
// on the host once per new t and uploads the table; the device never
// evaluates incomplete beta/gamma functions.  The numerics follow the
// reference's published algorithms operation for operation so the table
// matches the reference's memoised critical_value() bit for bit:
//   series / continued fraction for P(a, x)   special_functions.cpp:12-49
//   Lentz continued fraction for I_x(a, b)    special_functions.cpp:53-83
//   bisection quantile inversion              special_functions.cpp:88-102
//   chi-squared limit for d2 > 2e7            special_functions.cpp:150-160
// Compiled for the default x86-64 target (no FMA) like the reference.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>

#include "fppm_gpu.h"

namespace fppm_b200 {
namespace {

constexpr int kIterCap = 500;
const double kEpsilon = std::numeric_limits<double>::epsilon();
const double kTiny = std::numeric_limits<double>::min() / std::numeric_limits<double>::epsilon();

double lower_gamma_series(double a, double x) {
  double ap = a, total = 1.0 / a, term = total;
  for (int n = 0; n < kIterCap; ++n) {
    ap += 1.0;
    term *= x / ap;
    total += term;
    if (std::fabs(term) < std::fabs(total) * kEpsilon) break;
  }
  return total * std::exp(-x + a * std::log(x) - std::lgamma(a));
}

double upper_gamma_fraction(double a, double x) {
  double b = x + 1.0 - a, c = 1.0 / kTiny, d = 1.0 / b, h = d;
  for (int n = 1; n <= kIterCap; ++n) {
    const double an = -n * (n - a);
    b += 2.0;
    d = an * d + b;
    if (std::fabs(d) < kTiny) d = kTiny;
    c = b + an / c;
    if (std::fabs(c) < kTiny) c = kTiny;
    d = 1.0 / d;
    const double step = d * c;
    h *= step;
    if (std::fabs(step - 1.0) < kEpsilon) break;
  }
  return h * std::exp(-x + a * std::log(x) - std::lgamma(a));
}

double beta_fraction(double a, double b, double x) {
  const double qab = a + b, qap = a + 1.0, qam = a - 1.0;
  double c = 1.0, d = 1.0 - qab * x / qap;
  if (std::fabs(d) < kTiny) d = kTiny;
  d = 1.0 / d;
  double h = d;
  for (int m = 1; m <= kIterCap; ++m) {
    const int m2 = 2 * m;
    double coef = m * (b - m) * x / ((qam + m2) * (a + m2));
    d = 1.0 + coef * d;
    if (std::fabs(d) < kTiny) d = kTiny;
    c = 1.0 + coef / c;
    if (std::fabs(c) < kTiny) c = kTiny;
    d = 1.0 / d;
    h *= d * c;
    coef = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2));
    d = 1.0 + coef * d;
    if (std::fabs(d) < kTiny) d = kTiny;
    c = 1.0 + coef / c;
    if (std::fabs(c) < kTiny) c = kTiny;
    d = 1.0 / d;
    const double step = d * c;
    h *= step;
    if (std::fabs(step - 1.0) < kEpsilon) break;
  }
  return h;
}

double reg_lower_gamma(double a, double x) {
  if (x == 0.0) return 0.0;
  return x < a + 1.0 ? lower_gamma_series(a, x) : 1.0 - upper_gamma_fraction(a, x);
}

double reg_inc_beta(double a, double b, double x) {
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  const double front = std::exp(std::lgamma(a + b) - std::lgamma(a) - std::lgamma(b) +
                                a * std::log(x) + b * std::log1p(-x));
  if (x < (a + 1.0) / (a + b + 2.0)) return front * beta_fraction(a, b, x) / a;
  return 1.0 - front * beta_fraction(b, a, 1.0 - x) / b;
}

double chi2_cdf(double x, double df) { return x <= 0.0 ? 0.0 : reg_lower_gamma(0.5 * df, 0.5 * x); }

double f_cdf(double x, double d1, double d2) {
  if (x <= 0.0) return 0.0;
  if (d2 > 2e7) return reg_lower_gamma(0.5 * d1, 0.5 * d1 * x);
  return reg_inc_beta(0.5 * d1, 0.5 * d2, d1 * x / (d1 * x + d2));
}

template <typename Cdf>
double bisect(const Cdf &cdf, double p, double lo, double hi) {
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (mid == lo || mid == hi) break;
    if (cdf(mid) < p)
      lo = mid;
    else
      hi = mid;
    if (hi - lo <= 1e-15 * std::max(1.0, lo)) break;
  }
  return 0.5 * (lo + hi);
}

}  // namespace

double host_f_quantile(double p, double d1, double d2, int *status) {
  if (!(p > 0.0 && p < 1.0) || !(d1 > 0.0) || !(d2 > 0.0)) {
    if (status) *status = FPPM_ERR_INVALID_ARGUMENT;
    return 0.0;
  }
  double hi = 16.0;
  while (f_cdf(hi, d1, d2) < p) hi *= 4.0;
  return bisect([&](double x) { return f_cdf(x, d1, d2); }, p, 0.0, hi);
}

double host_chi2_quantile(double p, double df, int *status) {
  if (!(p > 0.0 && p < 1.0) || !(df > 0.0)) {
    if (status) *status = FPPM_ERR_INVALID_ARGUMENT;
    return 0.0;
  }
  double hi = df + 10.0 * std::sqrt(2.0 * df) + 10.0;
  while (chi2_cdf(hi, df) < p) hi *= 2.0;
  return bisect([&](double x) { return chi2_cdf(x, df); }, p, 0.0, hi);
}

// gather.cpp:11-13
double host_schedule_radius(double base, double alpha, uint64_t i) {
  return base * std::sqrt(std::pow(static_cast<double>(i), alpha - 1.0));
}

}  // namespace fppm_b200

namespace fppm_b200 {

// ---- host restatements used by the reference-shaped C++ wrapper
// gather.cpp:15-33 (glibc atan2, as the reference build): 0 ok, 1 invalid
// argument (bin counts), 2 domain error (outside the disk)
int host_sector_index(double u, double v, double radius, int na, int ns, int *status) {
  *status = 0;
  if (na < 1 || ns < 1) {
    *status = 1;
    return 0;
  }
  const double r2 = radius * radius;
  const double d2 = u * u + v * v;
  if (d2 > r2 * (1.0 + 1e-9)) {
    *status = 2;
    return 0;
  }
  int a = static_cast<int>(static_cast<double>(na) * d2 / r2);
  a = a < na - 1 ? a : na - 1;
  const double two_pi = 6.283185307179586476925286766559;
  double theta = std::atan2(v, u);
  if (theta < 0.0) theta += two_pi;
  int s = static_cast<int>(static_cast<double>(ns) * theta / two_pi);
  s = s < ns - 1 ? s : ns - 1;
  return a * ns + s;
}

// frame.cpp:5-14 (Duff et al. branchless basis)
void host_build_frame(const double n[3], double u[3], double v[3]) {
  const double sign = std::copysign(1.0, n[2]);
  const double a = -1.0 / (sign + n[2]);
  const double b = n[0] * n[1] * a;
  u[0] = 1.0 + sign * n[0] * n[0] * a;
  u[1] = sign * b;
  u[2] = -sign * n[0];
  v[0] = b;
  v[1] = sign + n[1] * n[1] * a;
  v[2] = -n[1];
}

}  // namespace fppm_b200
