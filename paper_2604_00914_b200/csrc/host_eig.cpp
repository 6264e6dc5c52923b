// Small symmetric eigensolver on the host (cyclic Jacobi), for the Lanczos
// tridiagonal (<= lanczos_steps, default 40; proj/src/lanczos.cpp:61-69). The
// projected Rayleigh-Ritz problems go to cuSOLVER syevd on the device.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "dense.hpp"

namespace adp {

std::vector<double> host_sym_eig(std::vector<double>& a, int p, std::vector<double>& z) {
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(i) + static_cast<size_t>(j) * p]; };
  std::vector<double> v(static_cast<size_t>(p) * p, 0.0);
  auto V = [&](int i, int j) -> double& { return v[static_cast<size_t>(i) + static_cast<size_t>(j) * p]; };
  for (int i = 0; i < p; ++i) V(i, i) = 1.0;
  // symmetrise as sym_eig does ((B + B^T) / 2, dense_kernels.cpp:34)
  for (int j = 0; j < p; ++j)
    for (int i = j + 1; i < p; ++i) A(i, j) = A(j, i) = 0.5 * (A(i, j) + A(j, i));
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int j = 0; j < p; ++j)
      for (int i = 0; i < p; ++i) {
        tot += A(i, j) * A(i, j);
        if (i != j) off += A(i, j) * A(i, j);
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int pi = 0; pi < p - 1; ++pi)
      for (int qi = pi + 1; qi < p; ++qi) {
        const double apq = A(pi, qi);
        if (apq == 0.0) continue;
        const double app = A(pi, pi), aqq = A(qi, qi);
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < p; ++k) {
          const double akp = A(k, pi), akq = A(k, qi);
          A(k, pi) = c * akp - s * akq;
          A(k, qi) = s * akp + c * akq;
        }
        for (int k = 0; k < p; ++k) {
          const double apk = A(pi, k), aqk = A(qi, k);
          A(pi, k) = c * apk - s * aqk;
          A(qi, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < p; ++k) {
          const double vkp = V(k, pi), vkq = V(k, qi);
          V(k, pi) = c * vkp - s * vkq;
          V(k, qi) = s * vkp + c * vkq;
        }
      }
  }
  std::vector<int> order(p);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int x, int y) { return A(x, x) < A(y, y); });
  std::vector<double> w(p);
  z.assign(static_cast<size_t>(p) * p, 0.0);
  for (int j = 0; j < p; ++j) {
    w[j] = A(order[j], order[j]);
    for (int i = 0; i < p; ++i) z[static_cast<size_t>(i) + static_cast<size_t>(j) * p] = V(i, order[j]);
  }
  return w;
}

}  // namespace adp
