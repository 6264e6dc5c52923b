// C entry points over the REFERENCE's own filter-path sources, compiled where they lie under
// /root/reference/proj (this file includes them; nothing is copied) against oracle/eigen_standin (Eigen is
// not in this image: the stand-in covers the elementwise subset this path uses, see its header).
// Output: oracle/_ref/libadapoly_ref.so (git-ignored). Test infrastructure: tests/test_ref_build.py checks
// the oracle restatement (oracle/oracle.cpp) bit for bit against it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "adapoly/cheb_filter.hpp"
#include "adapoly/csr_matrix.hpp"
#include "adapoly/philox.hpp"
#include "adapoly/tiled_matrix.hpp"

using namespace adapoly;

namespace {
CsrMatrixd make_csr(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci, const double* v) {
  CsrMatrixd a;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.row_ptr.assign(rp, rp + n_rows + 1);
  a.col_idx.assign(ci, ci + rp[n_rows]);
  a.values.assign(v, v + rp[n_rows]);
  return a;
}
Matrixd make_matrix(const double* p, int64_t r, int64_t c) {
  Matrixd m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}
ChebFilter make_filter(const double* coeffs, int k_max, double l1, double l2) {
  ChebFilter f;
  f.k_max = k_max;
  f.l1 = l1;
  f.l2 = l2;
  f.coeffs.assign(coeffs, coeffs + k_max + 1);
  f.active_degree = k_max;
  return f;
}
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError&) {
    return 1;
  } catch (const DimensionError&) {
    return 2;
  } catch (const std::exception&) {
    return 9;
  }
}
}  // namespace

extern "C" {

// philox.hpp:92-109 (column-major n x q)
int ref_fill_gaussian(int64_t n, int64_t q, uint64_t seed, uint64_t stream, double* out) {
  return guarded([&] {
    Matrixd m(n, q);
    fill_gaussian(m, seed, stream);
    std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(n * q));
  });
}
int ref_fill_rademacher(int64_t n, int64_t q, uint64_t seed, uint64_t stream, double* out) {
  return guarded([&] {
    Matrixd m(n, q);
    fill_rademacher(m, seed, stream);
    std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(n * q));
  });
}

// cheb_filter.cpp:64-97; damping 0 lanczos, 1 jackson; out: coeffs[k+1], params {l1, l2, alpha, beta}
int ref_build_filter(double a, double b, double lmin, double lmax, int k, double m, int damping, double* coeffs,
                     double* params) {
  return guarded([&] {
    const ChebFilter f =
        build_filter(a, b, SpectrumBounds{lmin, lmax}, k, m, damping ? DampingKind::jackson : DampingKind::lanczos);
    std::memcpy(coeffs, f.coeffs.data(), sizeof(double) * f.coeffs.size());
    params[0] = f.l1;
    params[1] = f.l2;
    params[2] = f.alpha;
    params[3] = f.beta;
  });
}

// csr_to_tiled (tiled_matrix.hpp:58-94) + to_block_layout + maspmm (:184-210) + from_block_layout; C in/out
int ref_maspmm(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci, const double* v, int64_t t_i,
               int64_t t_k, const double* b, int64_t k, double* c) {
  return guarded([&] {
    const TiledMatrixd t = csr_to_tiled(make_csr(n_rows, n_cols, rp, ci, v), t_i, t_k);
    const Matrixd bm = make_matrix(b, n_cols, k), cm = make_matrix(c, n_rows, k);
    const BlockMatrixd bb = to_block_layout<double>(bm, t_k);
    BlockMatrixd cb = to_block_layout<double>(cm, t_k);
    maspmm(t, bb, cb);
    const Matrixd out = from_block_layout(cb);
    std::memcpy(c, out.data(), sizeof(double) * static_cast<size_t>(n_rows * k));
  });
}

// clenshaw_apply (cheb_filter.cpp:129-179) on csr_to_tiled(A, t_i, t_k); x, y column-major
int ref_clenshaw_apply(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t t_i, int64_t t_k,
                       const double* coeffs, int k_max, double l1, double l2, const double* x, int64_t q, int degree,
                       double* y, int64_t* spmv_count) {
  return guarded([&] {
    const TiledMatrixd t = csr_to_tiled(make_csr(n, n, rp, ci, v), t_i, t_k);
    const ChebFilter f = make_filter(coeffs, k_max, l1, l2);
    const Matrixd xm = make_matrix(x, n, q);
    const Matrixd out = clenshaw_apply(f, t, xm, degree, spmv_count);
    std::memcpy(y, out.data(), sizeof(double) * static_cast<size_t>(out.rows() * out.cols()));
  });
}

// csr_spmv (csr_matrix.hpp:122-134), naive_spmm (:138-147)
int ref_csr_spmv(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci, const double* v,
                 const double* x, double* y) {
  return guarded([&] {
    Vectord xv(n_cols);
    std::memcpy(xv.data(), x, sizeof(double) * static_cast<size_t>(n_cols));
    const Vectord out = csr_spmv(make_csr(n_rows, n_cols, rp, ci, v), xv);
    std::memcpy(y, out.data(), sizeof(double) * static_cast<size_t>(n_rows));
  });
}
int ref_naive_spmm(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci, const double* v,
                   const double* b, int64_t k, double* c) {
  return guarded([&] {
    const Matrixd out = naive_spmm(make_csr(n_rows, n_cols, rp, ci, v), make_matrix(b, n_cols, k));
    std::memcpy(c, out.data(), sizeof(double) * static_cast<size_t>(n_rows * k));
  });
}

// eval_filter_scalar (cheb_filter.cpp:99-127), initial_degree (:181-187), adaptive_degree (:189-219)
int ref_eval_filter(const double* coeffs, int k_max, double l1, double l2, const double* x, int64_t n, int degree,
                    double* out, int64_t* clamped) {
  return guarded([&] {
    const ChebFilter f = make_filter(coeffs, k_max, l1, l2);
    Vectord xv(n);
    std::memcpy(xv.data(), x, sizeof(double) * static_cast<size_t>(n));
    index_t c = 0;
    const Vectord r = eval_filter_scalar(f, xv, degree, &c);
    std::memcpy(out, r.data(), sizeof(double) * static_cast<size_t>(n));
    if (clamped) *clamped = c;
  });
}
// CPU baseline timing: `steps` middle Clenshaw steps (cheb_filter.cpp:167-173) on block-layout operands.
// csr_to_tiled, BlockMatrix, set_zero and maspmm are the reference's own code (tiled_matrix.hpp: plain
// C++ + OpenMP, no Eigen inside); the array update is written as the single pass Eigen's expression
// template generates for `v = 2 l1 aw + 2 l2 w - v + c y` (one thread, one loop over the block) -- the
// stand-in's eager temporaries would make it several passes and the reference look slower than it is.
void* ref_tiled_create(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t t_i, int64_t t_k) {
  try {
    return new TiledMatrixd(csr_to_tiled(make_csr(n, n, rp, ci, v), t_i, t_k));
  } catch (const std::exception&) {
    return nullptr;
  }
}
void ref_tiled_destroy(void* h) { delete static_cast<TiledMatrixd*>(h); }
int ref_bench_clenshaw_steps(const void* h, int64_t q, int steps, double* seconds, double* checksum) {
  return guarded([&] {
    const TiledMatrixd& t = *static_cast<const TiledMatrixd*>(h);
    const index_t n = t.n_rows;
    const index_t t_k = t.t_k;
    BlockMatrixd y(n, q, t_k), w(n, q, t_k), vv(n, q, t_k), aw(n, q, t_k);
    const Philox4x32 rng(7, 7);
    const index_t sz = y.size();
#pragma omp parallel for schedule(static)
    for (index_t i = 0; i < sz; ++i) {
      y.data()[i] = rng.uniform(static_cast<std::uint64_t>(i)) - 0.5;
      w.data()[i] = 0.5 * y.data()[i];
      vv.data()[i] = 0.25 * y.data()[i];
    }
    const double two_l1 = 0.25, two_l2 = -0.5, cj = 0.01;
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s) {
      aw.set_zero();
      maspmm(t, w, aw);
      double* vd = vv.data();
      const double* ad = aw.data();
      const double* wd = w.data();
      const double* yd = y.data();
      for (index_t i = 0; i < sz; ++i) vd[i] = two_l1 * ad[i] + two_l2 * wd[i] - vd[i] + cj * yd[i];
      std::swap(vv, w);
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double cs = 0.0;
    for (index_t i = 0; i < sz; i += 97) cs += w.data()[i];
    *checksum = cs;
  });
}

int ref_initial_degree(double alpha, double beta, double c, int* out) {
  return guarded([&] { *out = initial_degree(alpha, beta, c); });
}
int ref_adaptive_degree(const double* coeffs, int k_max, double l1, double l2, const double* ritz, int64_t p,
                        int64_t e_i, double tau_a, int* out) {
  return guarded([&] {
    const ChebFilter f = make_filter(coeffs, k_max, l1, l2);
    Vectord rv(p);
    std::memcpy(rv.data(), ritz, sizeof(double) * static_cast<size_t>(p));
    *out = adaptive_degree(f, rv, e_i, tau_a);
  });
}
}
