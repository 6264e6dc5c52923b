// Host-side filter construction and degree logic (product path).
//
// These are O(k) / O(k p log p) scalar computations that stay on the host
// (SURVEY.md 8a rows a5-a6): the device only ever receives the coefficient
// array and per-step scalars. Restated from proj/src/cheb_filter.cpp with the
// reference's exact expression forms, so the coefficient bits -- and hence the
// filtered blocks -- match the reference.
#include <algorithm>
#include <cmath>
#include <functional>
#include <numbers>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

namespace {
constexpr double kPi = std::numbers::pi;
}

// chebyshev_step_coeffs (cheb_filter.cpp:21-37)
std::vector<double> step_coeffs(double alpha, double beta, int k) {
  if (!(0.0 <= beta && beta < alpha && alpha <= kPi))
    fail(ADP_ERR_CONFIG, "chebyshev_step_coeffs: need 0 <= beta < alpha <= pi");
  if (k < 0) fail(ADP_ERR_CONFIG, "chebyshev_step_coeffs: negative degree");
  std::vector<double> c(static_cast<size_t>(k) + 1);
  c[0] = (alpha - beta) / kPi;
  // alpha / beta equal to the double nearest pi mean exactly pi (sin(j pi) = 0).
  const bool alpha_pi = alpha == kPi;
  const bool beta_pi = beta == kPi;
  for (int j = 1; j <= k; ++j) {
    const double sa = alpha_pi ? 0.0 : std::sin(j * alpha);
    const double sb = beta_pi ? 0.0 : std::sin(j * beta);
    c[j] = (2.0 / kPi) * (sa - sb) / j;
  }
  return c;
}

// lanczos_damping (cheb_filter.cpp:39-49): d_j = (sin u / u)^m, u = j pi / (k+1)
std::vector<double> lanczos_damping(int k, double m) {
  if (k < 1) fail(ADP_ERR_CONFIG, "lanczos_damping: degree must be >= 1");
  if (m < 0.0) fail(ADP_ERR_CONFIG, "lanczos_damping: exponent must be >= 0");
  std::vector<double> d(static_cast<size_t>(k) + 1);
  d[0] = 1.0;
  for (int j = 1; j <= k; ++j) {
    const double u = j * kPi / (k + 1);
    d[j] = std::pow(std::sin(u) / u, m);
  }
  return d;
}

// jackson_damping (cheb_filter.cpp:51-61)
std::vector<double> jackson_damping(int k) {
  if (k < 1) fail(ADP_ERR_CONFIG, "jackson_damping: degree must be >= 1");
  std::vector<double> d(static_cast<size_t>(k) + 1);
  d[0] = 1.0;
  const double h = kPi / (k + 2);
  for (int j = 1; j <= k; ++j)
    d[j] = ((k + 2 - j) * std::sin(h) * std::cos(j * h) + std::cos(h) * std::sin(j * h)) / ((k + 2) * std::sin(h));
  return d;
}

// ChebFilter::map_clamped (cheb_filter.hpp:55-62)
double map_clamped(const adp_filter_info& f, double x, bool* clamped) {
  const double t = f.l1 * x + f.l2;
  if (t < -1.0 || t > 1.0) {
    if (clamped) *clamped = true;
    return t < -1.0 ? -1.0 : 1.0;
  }
  return t;
}

}  // namespace adp

using adp::Error;

namespace {
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

adp_status adp_step_coeffs(double alpha, double beta, int32_t k, double* out) {
  return guarded([&] {
    const auto c = adp::step_coeffs(alpha, beta, k);
    std::copy(c.begin(), c.end(), out);
  });
}

adp_status adp_lanczos_damping(int32_t k, double m, double* out) {
  return guarded([&] {
    const auto d = adp::lanczos_damping(k, m);
    std::copy(d.begin(), d.end(), out);
  });
}

adp_status adp_jackson_damping(int32_t k, double* out) {
  return guarded([&] {
    const auto d = adp::jackson_damping(k);
    std::copy(d.begin(), d.end(), out);
  });
}

// build_filter (cheb_filter.cpp:63-94)
adp_status adp_build_filter(double a, double b, double lambda_min, double lambda_max, int32_t k, double m,
                            adp_damping damping, adp_filter_info* f, double* coeffs) {
  return guarded([&] {
    if (!std::isfinite(lambda_min) || !std::isfinite(lambda_max) || !(lambda_min < lambda_max))
      adp::fail(ADP_ERR_CONFIG, "build_filter: invalid spectrum bounds");
    if (!(lambda_min <= a && a < b && b <= lambda_max))
      adp::fail(ADP_ERR_CONFIG, "build_filter: target interval must lie inside the spectrum bounds");
    if (k < 1) adp::fail(ADP_ERR_CONFIG, "build_filter: degree must be >= 1");
    if (m < 0.0) adp::fail(ADP_ERR_CONFIG, "build_filter: damping exponent must be >= 0");
    adp_filter_info g{};
    g.interval_a = a;
    g.interval_b = b;
    g.k_max = k;
    g.m = m;
    g.lambda_min = lambda_min;
    g.lambda_max = lambda_max;
    const double span = lambda_max - lambda_min;
    g.l1 = 2.0 / span;
    g.l2 = -(lambda_max + lambda_min) / span;
    g.alpha = std::acos(adp::map_clamped(g, a, nullptr));
    g.beta = std::acos(adp::map_clamped(g, b, nullptr));
    if (!(g.alpha > g.beta)) adp::fail(ADP_ERR_CONFIG, "build_filter: interval collapses under the spectral map");
    const auto c = adp::step_coeffs(g.alpha, g.beta, k);
    const auto d = damping == ADP_DAMP_LANCZOS ? adp::lanczos_damping(k, m) : adp::jackson_damping(k);
    for (size_t j = 0; j < c.size(); ++j) coeffs[j] = c[j] * d[j];
    g.active_degree = k;
    *f = g;
  });
}

// eval_filter_scalar (cheb_filter.cpp:96-127)
adp_status adp_eval_filter(const adp_filter_info* f, const double* coeffs, const double* x, int64_t n,
                           int32_t degree, double* out, int64_t* clamped) {
  return guarded([&] {
    if (degree < 0 || degree > f->k_max) adp::fail(ADP_ERR_CONFIG, "eval_filter_scalar: degree out of range");
    int64_t nc = 0;
    for (int64_t i = 0; i < n; ++i) {
      bool c = false;
      const double t = adp::map_clamped(*f, x[i], &c);
      nc += c ? 1 : 0;
      double acc = coeffs[0];
      if (degree >= 1) {
        double t_prev = 1.0, t_cur = t;
        acc += coeffs[1] * t_cur;
        for (int j = 2; j <= degree; ++j) {
          const double t_next = 2.0 * t * t_cur - t_prev;
          acc += coeffs[j] * t_next;
          t_prev = t_cur;
          t_cur = t_next;
        }
      }
      out[i] = acc;
    }
    if (clamped) *clamped += nc;
  });
}

// initial_degree (cheb_filter.cpp:181-187)
adp_status adp_initial_degree(double alpha, double beta, double c, int32_t* out) {
  return guarded([&] {
    const double width = alpha - beta;
    if (!(width > 0.0)) adp::fail(ADP_ERR_CONFIG, "initial_degree: need alpha > beta");
    if (!(c > width)) adp::fail(ADP_ERR_CONFIG, "initial_degree: constant must exceed alpha - beta");
    const int k1 = static_cast<int>(std::ceil(c / width)) - 1;
    *out = std::max(k1, 1);
  });
}

// adaptive_degree (cheb_filter.cpp:189-219)
adp_status adp_adaptive_degree(const adp_filter_info* f, const double* coeffs, const double* ritz, int64_t p,
                               int64_t e_i, double tau_a, int32_t* out) {
  return guarded([&] {
    if (p < 1) adp::fail(ADP_ERR_CONFIG, "adaptive_degree: empty Ritz set");
    if (e_i < 1 || e_i > p) adp::fail(ADP_ERR_CONFIG, "adaptive_degree: in-interval count out of range");
    if (!(tau_a > 0.0)) adp::fail(ADP_ERR_CONFIG, "adaptive_degree: threshold must be positive");
    const int floor_degree = std::min(3, f->k_max);
    std::vector<double> t(p), h_prev(p, 1.0), h_cur(p), gamma(p, coeffs[0]), mags(p), h_next(p);
    for (int64_t i = 0; i < p; ++i) t[i] = adp::map_clamped(*f, ritz[i], nullptr);
    h_cur = t;
    for (int j = 1; j <= f->k_max; ++j) {
      for (int64_t i = 0; i < p; ++i) gamma[i] += coeffs[j] * h_cur[i];
      for (int64_t i = 0; i < p; ++i) mags[i] = std::abs(gamma[i]);
      // Only the e_i-th largest and the smallest magnitudes are needed.
      std::sort(mags.begin(), mags.end(), std::greater<double>());
      const double denom = mags[e_i - 1];
      const double num = mags[p - 1];
      if (denom > 0.0 && num / denom < tau_a) {
        *out = std::min(std::max(j, floor_degree), f->k_max);
        return;
      }
      for (int64_t i = 0; i < p; ++i) h_next[i] = 2.0 * t[i] * h_cur[i] - h_prev[i];
      std::swap(h_prev, h_cur);
      std::swap(h_cur, h_next);
    }
    *out = f->k_max;
  });
}

}  // extern "C"
