// C++ caller of the C-ABI (include/adp.h), the way the reference code base
// would bind it: builds a 3D 7-point operator, builds the
// filter with adp_build_filter, applies clenshaw_apply through the host API on
// an Eigen-style column-major block, and checks the result BITWISE against the
// CPU oracle's restatement of the reference (liboracle.so, test infrastructure),
// then runs adp_solve on a diagonal operator and checks the eigenvalues.
// Exit code 0 on success. Built by __graft_entry__.build(); run by
// tests/test_gpu_cpp.py on the GPU box.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "adp.h"

extern "C" {
// oracle.cpp (test infrastructure)
struct orc_csr;
struct orc_tiled;
orc_csr* orc_csr_wrap(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci, const double* v);
int orc_tiled_create(const orc_csr* a, int64_t ti, int64_t tk, orc_tiled** out);
int orc_clenshaw_apply(const double* coeffs, int k_max, double l1, double l2, const orc_tiled* a, const double* x,
                       int64_t n, int64_t q, int degree, double* out, int64_t* spmv_count);
void orc_fill_gaussian(double* out, int64_t n, int64_t q, uint64_t seed, uint64_t stream);
}

#define CHECK(x)                                                                         \
  do {                                                                                   \
    adp_status s__ = (x);                                                                \
    if (s__ != ADP_OK) {                                                                 \
      std::fprintf(stderr, "%s failed: %d %s\n", #x, (int)s__, adp_last_error_message()); \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

int main() {
  const int nx = 24;
  const int64_t n = int64_t{nx} * nx * nx;
  std::vector<int64_t> rp{0}, ci;
  std::vector<double> val;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t x = r % nx, y = (r / nx) % nx, z = r / (nx * nx);
    const int64_t nb[7] = {z > 0 ? r - nx * nx : -1, y > 0 ? r - nx : -1, x > 0 ? r - 1 : -1, r,
                           x < nx - 1 ? r + 1 : -1, y < nx - 1 ? r + nx : -1, z < nx - 1 ? r + nx * nx : -1};
    for (int k = 0; k < 7; ++k) {
      if (nb[k] < 0) continue;
      ci.push_back(nb[k]);
      val.push_back(nb[k] == r ? 6.0 + 0.001 * static_cast<double>(r % 97) : -1.0);
    }
    rp.push_back(static_cast<int64_t>(ci.size()));
  }
  // filter: build_filter (cheb_filter.cpp:63-94)
  const int k = 60;
  adp_filter_info f{};
  std::vector<double> coeffs(k + 1);
  CHECK(adp_build_filter(5.9, 6.1, -0.1, 12.2, k, 0.5, ADP_DAMP_LANCZOS, &f, coeffs.data()));
  int32_t k1 = 0;
  CHECK(adp_initial_degree(f.alpha, f.beta, 1.4, &k1));

  adp_ctx* ctx = nullptr;
  CHECK(adp_ctx_create(0, &ctx));
  adp_csr* a = nullptr;
  CHECK(adp_csr_create(ctx, n, n, rp.data(), ci.data(), val.data(), ADP_F64, &a));

  const int64_t q = 10;
  std::vector<double> x(n * q), y(n * q), want(n * q);
  orc_fill_gaussian(x.data(), n, q, 5, 0);
  int64_t spmv = 0;
  CHECK(adp_filter_apply(ctx, a, coeffs.data(), k, f.l1, f.l2, k, x.data(), n, n, q, ADP_COL_MAJOR, y.data(), n,
                         &spmv));
  orc_csr* oc = orc_csr_wrap(n, n, rp.data(), ci.data(), val.data());
  orc_tiled* ot = nullptr;
  if (orc_tiled_create(oc, 256, 64, &ot) != 0) return 2;
  int64_t spmv2 = 0;
  if (orc_clenshaw_apply(coeffs.data(), k, f.l1, f.l2, ot, x.data(), n, q, k, want.data(), &spmv2) != 0) return 2;
  if (std::memcmp(y.data(), want.data(), y.size() * sizeof(double)) != 0 || spmv != spmv2) {
    std::fprintf(stderr, "clenshaw_apply through the C-ABI differs from the oracle\n");
    return 3;
  }
  // error mapping: degree out of range -> ConfigError
  if (adp_filter_apply(ctx, a, coeffs.data(), k, f.l1, f.l2, k + 1, x.data(), n, n, q, ADP_COL_MAJOR, y.data(), n,
                       nullptr) != ADP_ERR_CONFIG)
    return 4;

  // solve on diag(1..100), interval [10.5, 20.5] -> 11..20 (test_eigensolver.cpp:168-192)
  std::vector<int64_t> drp(101), dci(100);
  std::vector<double> dv(100);
  for (int i = 0; i < 100; ++i) {
    drp[i + 1] = i + 1;
    dci[i] = i;
    dv[i] = i + 1.0;
  }
  adp_csr* d = nullptr;
  CHECK(adp_csr_create(ctx, 100, 100, drp.data(), dci.data(), dv.data(), ADP_F64, &d));
  adp_solver_config cfg;
  adp_solver_config_default(&cfg);
  cfg.interval_a = 10.5;
  cfg.interval_b = 20.5;
  cfg.rng_seed = 7;
  adp_solve_result* res = nullptr;
  CHECK(adp_solve(ctx, d, &cfg, &res));
  adp_solve_summary s{};
  CHECK(adp_solve_summary_get(res, &s));
  std::vector<double> ev(s.n_eigs);
  CHECK(adp_solve_eigenpairs(res, ev.data(), nullptr, 0));
  if (!s.converged || s.n_eigs != 10) return 5;
  for (int i = 0; i < 10; ++i)
    if (std::abs(ev[i] - (11.0 + i)) > 1e-9 * (11.0 + i)) return 6;
  CHECK(adp_solve_result_destroy(res));
  CHECK(adp_csr_destroy(d));
  CHECK(adp_csr_destroy(a));
  CHECK(adp_ctx_destroy(ctx));
  std::printf("capi_from_cpp ok: n=%lld q=%lld degree=%d bitwise==oracle, spmv=%lld; solve 10 eigenpairs\n",
              static_cast<long long>(n), static_cast<long long>(q), k, static_cast<long long>(spmv));
  return 0;
}
