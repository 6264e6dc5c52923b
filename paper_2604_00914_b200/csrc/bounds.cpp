// Truncation-error bounds of the damped Chebyshev step filter (host).
//
// Restates the reference's filter diagnostics (proj/src/filter_bounds.cpp,
// declared in proj/include/adapoly/filter_bounds.hpp:8-30): the reciprocal-sine
// sum J(theta), the damping constant C_m, the pointwise undamped / damped
// bounds and the projector bound used by `inspect-filter`
// (proj/src/cli.cpp:198-235). Same formulas, same error behaviour
// (ConfigError -> ADP_ERR_CONFIG); C_m is computed here by double-exponential
// (tanh-sinh) quadrature, which handles the integrable endpoint singularity at
// pi for m < 1 without the reference's change of variables, to ~1e-13.
#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <mutex>
#include <numbers>

#include "adp_internal.hpp"

namespace {

using adp::Error;
using adp::fail;
constexpr double kPi = std::numbers::pi;

double inv_abs_sin(double x) {
  const double s = std::fabs(std::sin(x));
  return s == 0.0 ? std::numeric_limits<double>::infinity() : 1.0 / s;
}

double sinc(double u) { return u == 0.0 ? 1.0 : std::sin(u) / u; }

double j_theta(double theta, double alpha, double beta) {
  const double plus = inv_abs_sin(0.5 * (alpha + beta)), minus = inv_abs_sin(0.5 * (alpha - beta));
  if (theta == alpha) return inv_abs_sin(alpha) + plus + minus;
  if (theta == beta) return inv_abs_sin(beta) + plus + minus;
  return inv_abs_sin(0.5 * (theta + alpha)) + inv_abs_sin(0.5 * (theta - alpha)) + inv_abs_sin(0.5 * (theta + beta)) +
         inv_abs_sin(0.5 * (theta - beta));
}

// Integrand of C_m at u = pi - s (both given, so neither end loses digits):
// sinc(u)^(m-1) * (sin u - u cos u) / u^3.
double cm_integrand(double u, double s, double m) {
  double g;
  if (u < 0.25) {  // (sin u - u cos u) / u^3 = 1/3 - u^2/30 + u^4/840 - u^6/45360 + ...
    const double u2 = u * u;
    g = 1.0 / 3.0 - u2 / 30.0 + u2 * u2 / 840.0 - u2 * u2 * u2 / 45360.0 + u2 * u2 * u2 * u2 / 3991680.0;
  } else {
    const double sn = std::sin(s), cs = -std::cos(s);  // sin u, cos u through s
    g = (sn - u * cs) / (u * u * u);
  }
  const double sc = u < 0.25 ? sinc(u) : std::sin(s) / u;
  return std::pow(sc, m - 1.0) * g;
}

// C_m = int_0^pi (sin u)^(m-1) (sin u - u cos u) / u^(m+2) du by tanh-sinh:
// u = (pi/2)(1 + tanh(pi/2 sinh t)), halving the step until two levels agree.
double c_m_quadrature(double m) {
  const double half = 0.5 * kPi;
  auto term = [&](double t) {
    const double sh = half * std::sinh(t);
    const double e = std::exp(2.0 * sh);  // 1 - tanh(sh) = 2 / (1 + e), 1 + tanh(sh) = 2e / (1 + e)
    const double s = half * 2.0 / (1.0 + e);        // pi - u
    const double u = half * 2.0 * e / (1.0 + e);    // u
    if (!(s > 0.0) || !(u > 0.0) || !std::isfinite(e)) return 0.0;
    const double ch = std::cosh(sh);
    const double w = half * half * std::cosh(t) / (ch * ch);
    const double v = w * cm_integrand(u, s, m);
    return std::isfinite(v) ? v : 0.0;
  };
  const double tmax = 4.5;
  double h = 0.5;
  double sum = term(0.0);
  for (double t = h; t <= tmax; t += h) sum += term(t) + term(-t);
  double prev = sum * h;
  for (int level = 0; level < 12; ++level) {
    h *= 0.5;
    for (double t = h; t <= tmax; t += 2.0 * h) sum += term(t) + term(-t);
    const double cur = sum * h;
    if (std::fabs(cur - prev) <= 1e-14 * std::fabs(cur)) return cur;
    prev = cur;
  }
  return prev;
}

double c_m_constant(double m) {
  if (!(m > 0.0)) fail(ADP_ERR_CONFIG, "c_m_constant: exponent must be positive");
  static std::map<double, double> cache;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(m);
    if (it != cache.end()) return it->second;
  }
  const double v = c_m_quadrature(m);
  std::lock_guard<std::mutex> lock(mu);
  cache.emplace(m, v);
  return v;
}

double undamped_bound(double theta, int k, double alpha, double beta) {
  if (k < 1) fail(ADP_ERR_CONFIG, "undamped_bound: degree must be >= 1");
  return j_theta(theta, alpha, beta) / (kPi * (k + 1));
}

double damped_bound(double theta, int k_i, int k, double m, double alpha, double beta) {
  if (k_i < 1 || k_i > k) fail(ADP_ERR_CONFIG, "damped_bound: need 1 <= k_i <= k");
  if (m < 0.0) fail(ADP_ERR_CONFIG, "damped_bound: damping exponent must be >= 0");
  if (m == 0.0) return undamped_bound(theta, k_i, alpha, beta);
  const double j = j_theta(theta, alpha, beta);
  const double d = std::pow(sinc(k_i * kPi / (k + 1)), m);
  return d * j / (kPi * (k_i + 1)) + m * c_m_constant(m) * j / (k + 1) +
         m * kPi * (kPi - theta) / (3.0 * (k + 1) * (k + 1));
}

double projector_bound(const adp_filter_info& f, const double* thetas, int64_t count, int k_i) {
  if (count <= 0) fail(ADP_ERR_CONFIG, "projector_bound: empty eigenvalue angle list");
  if (k_i < 1 || k_i > f.k_max) fail(ADP_ERR_CONFIG, "projector_bound: need 1 <= k_i <= k_max");
  double js = 0.0;
  for (int64_t i = 0; i < count; ++i) js = std::max(js, j_theta(thetas[i], f.alpha, f.beta));
  const int k = f.k_max;
  if (f.m == 0.0) return js / (kPi * (k_i + 1));
  const double d = std::pow(sinc(k_i * kPi / (k + 1)), f.m);
  return d * js / (kPi * (k_i + 1)) + f.m * c_m_constant(f.m) * js / (k + 1) + f.m * kPi * kPi / (3.0 * (k + 1) * (k + 1));
}

template <class F>
adp_status guarded(F&& f) {
  try {
    f();
    return ADP_OK;
  } catch (const Error& e) {
    adp::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    adp::set_last_error(e.what());
    return ADP_ERR_RUNTIME;
  }
}

}  // namespace

extern "C" {

adp_status adp_j_theta(double theta, double alpha, double beta, double* out) {
  return guarded([&] { *out = j_theta(theta, alpha, beta); });
}

adp_status adp_c_m_constant(double m, double* out) {
  return guarded([&] { *out = c_m_constant(m); });
}

adp_status adp_undamped_bound(double theta, int32_t k, double alpha, double beta, double* out) {
  return guarded([&] { *out = undamped_bound(theta, k, alpha, beta); });
}

adp_status adp_damped_bound(double theta, int32_t k_i, int32_t k, double m, double alpha, double beta, double* out) {
  return guarded([&] { *out = damped_bound(theta, k_i, k, m, alpha, beta); });
}

adp_status adp_projector_bound(const adp_filter_info* f, const double* thetas, int64_t count, int32_t k_i,
                               double* out) {
  return guarded([&] {
    if (!f) fail(ADP_ERR_CONFIG, "projector_bound: null filter");
    *out = projector_bound(*f, thetas, count, k_i);
  });
}

}  // extern "C"
