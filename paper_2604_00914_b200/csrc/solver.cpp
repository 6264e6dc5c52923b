// The filtered-subspace-iteration driver on device-resident blocks: spectrum
// bounds (Lanczos), trace estimate, CholQR2, Rayleigh-Ritz, residuals,
// spurious-Ritz exclusion, locking. Host C++ orchestration mirroring
// proj/src/solver.cpp:119-360 and proj/src/lanczos.cpp:20-111; every n-sized
// operation runs on the GPU (the fused filter kernel, cuBLAS, cuSOLVER, our
// reduction kernels); only O(p) scalars (Ritz values, residual norms) and the
// Lanczos tridiagonal cross to the host per iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "adp_internal.hpp"
#include "dense.hpp"

namespace adp {

namespace {

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

struct DeviceBlock {
  double* ptr = nullptr;
  int64_t ld = 0;
  DeviceBlock() = default;
  DeviceBlock(int64_t n, int64_t cols) {
    ld = std::max<int64_t>(2, adp::block_ld(cols, false));
    const size_t bytes = static_cast<size_t>(std::max<int64_t>(n, 1)) * ld * 8;
    ADP_CUDA(cudaMalloc(&ptr, bytes));
    ADP_CUDA(cudaMemset(ptr, 0, bytes));
  }
  DeviceBlock(const DeviceBlock&) = delete;
  DeviceBlock& operator=(const DeviceBlock&) = delete;
  DeviceBlock(DeviceBlock&& o) noexcept : ptr(o.ptr), ld(o.ld) { o.ptr = nullptr; }
  DeviceBlock& operator=(DeviceBlock&& o) noexcept {
    std::swap(ptr, o.ptr);
    std::swap(ld, o.ld);
    return *this;
  }
  ~DeviceBlock() {
    if (ptr) cudaFree(ptr);
  }
};

struct DeviceVec {
  double* ptr = nullptr;
  explicit DeviceVec(int64_t n) { ADP_CUDA(cudaMalloc(&ptr, static_cast<size_t>(std::max<int64_t>(n, 1)) * 8)); }
  ~DeviceVec() {
    if (ptr) cudaFree(ptr);
  }
  DeviceVec(const DeviceVec&) = delete;
  DeviceVec& operator=(const DeviceVec&) = delete;
};

void sync(adp_ctx* ctx) { ADP_CUDA(cudaStreamSynchronize(ctx->stream)); }

// host column-major n x q -> device row-major block
void upload_colmajor(adp_ctx* ctx, const double* host, int64_t n, int64_t q, DeviceBlock& dst) {
  if (n == 0 || q == 0) return;
  void* staging = ctx->ws[5].get(static_cast<size_t>(n) * q * 8);
  ADP_CUDA(cudaMemcpyAsync(staging, host, static_cast<size_t>(n) * q * 8, cudaMemcpyHostToDevice, ctx->stream));
  launch_colmajor_to_rowmajor(ctx, staging, n, q, n, dst.ptr, dst.ld, 8);
  sync(ctx);
}

// device row-major (first q columns) -> host column-major n x q
void download_colmajor(adp_ctx* ctx, const double* src, int64_t ld, int64_t n, int64_t q, double* host) {
  if (n == 0 || q == 0) return;
  void* staging = ctx->ws[5].get(static_cast<size_t>(n) * q * 8);
  launch_rowmajor_to_colmajor(ctx, src, n, q, ld, staging, n, 8);
  ADP_CUDA(cudaMemcpyAsync(host, staging, static_cast<size_t>(n) * q * 8, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
}

struct LanczosRun {
  double lower = 0.0, upper = 0.0;
  bool early_breakdown = false;
};

// lanczos_pass (lanczos.cpp:20-77): basis is a device n x steps column-major panel.
LanczosRun lanczos_pass(adp_ctx* ctx, const adp_csr* a, int64_t steps, uint64_t seed, uint64_t draw_offset,
                        int64_t* spmv_count) {
  const int64_t n = a->n_rows;
  double* basis = nullptr;
  ADP_CUDA(cudaMalloc(&basis, static_cast<size_t>(n) * steps * 8));
  struct Free {
    double* p;
    ~Free() { cudaFree(p); }
  } guard{basis};
  DeviceVec w(n), h(steps);
  std::vector<double> v(n), alphas(steps), betas(steps);
  check_status(adp_philox_gaussian(seed, 1, draw_offset, n, v.data()));
  ADP_CUDA(cudaMemcpyAsync(basis, v.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  const double v0 = nrm2(ctx, basis, n, 1);
  scal(ctx, 1.0 / v0, basis, 1, n);
  double scale = 0.0, beta_res = 0.0;
  int64_t completed = 0;
  bool breakdown = false;
  for (int64_t j = 0; j < steps; ++j) {
    double* bj = basis + j * n;
    spmv(ctx, a, bj, w.ptr);
    if (spmv_count) ++*spmv_count;
    alphas[j] = dot(ctx, bj, w.ptr, n, 1, 1);
    axpy(ctx, -alphas[j], bj, 1, w.ptr, 1, n);
    if (j > 0) axpy(ctx, -betas[j - 1], basis + (j - 1) * n, 1, w.ptr, 1, n);
    for (int pass = 0; pass < 2; ++pass) {  // full reorthogonalisation (lanczos.cpp:44-45)
      gemv(ctx, true, n, j + 1, 1.0, basis, n, w.ptr, 1, 0.0, h.ptr, 1);
      gemv(ctx, false, n, j + 1, -1.0, basis, n, h.ptr, 1, 1.0, w.ptr, 1);
    }
    const double beta = nrm2(ctx, w.ptr, n, 1);
    betas[j] = beta;
    completed = j + 1;
    scale = std::max({scale, std::abs(alphas[j]), beta});
    if (beta <= scale * 1e-13) {
      beta_res = beta;
      breakdown = true;
      break;
    }
    if (j + 1 < steps) {
      ADP_CUDA(cudaMemcpyAsync(basis + (j + 1) * n, w.ptr, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      scal(ctx, 1.0 / beta, basis + (j + 1) * n, 1, n);
    } else {
      beta_res = beta;
    }
  }
  sync(ctx);
  const int p = static_cast<int>(completed);
  std::vector<double> tri(static_cast<size_t>(p) * p, 0.0), z;
  for (int j = 0; j < p; ++j) {
    tri[j + static_cast<size_t>(j) * p] = alphas[j];
    if (j + 1 < p) {
      tri[j + static_cast<size_t>(j + 1) * p] = betas[j];
      tri[j + 1 + static_cast<size_t>(j) * p] = betas[j];
    }
  }
  const std::vector<double> ev = host_sym_eig(tri, p, z);
  const double r_min = beta_res * std::abs(z[(p - 1) + static_cast<size_t>(0) * p]);
  const double r_max = beta_res * std::abs(z[(p - 1) + static_cast<size_t>(p - 1) * p]);
  LanczosRun run;
  run.lower = ev[0] - r_min;
  run.upper = ev[p - 1] + r_max;
  run.early_breakdown = breakdown && completed < steps;
  return run;
}

void validate_config(const adp_solver_config& c) {  // solver.cpp:22-38
  if (!(c.interval_a < c.interval_b)) fail(ADP_ERR_CONFIG, "solve: need interval_a < interval_b");
  if (!(c.tau_c > 0.0 && c.tau_c < 1.0)) fail(ADP_ERR_CONFIG, "solve: tau_c must lie in (0,1)");
  if (!(c.tau_a > 0.0 && c.tau_a < 1.0)) fail(ADP_ERR_CONFIG, "solve: tau_a must lie in (0,1)");
  if (!(c.mu >= 1.0)) fail(ADP_ERR_CONFIG, "solve: mu must be >= 1");
  if (c.m < 0.0) fail(ADP_ERR_CONFIG, "solve: damping exponent must be >= 0");
  if (!(c.c > 0.0)) fail(ADP_ERR_CONFIG, "solve: initial-degree constant must be positive");
  if (!(c.k_multiplier >= 1.0)) fail(ADP_ERR_CONFIG, "solve: k_multiplier must be >= 1");
  if (c.max_iter < 1) fail(ADP_ERR_CONFIG, "solve: max_iter must be >= 1");
  if (c.lanczos_steps < 2) fail(ADP_ERR_CONFIG, "solve: lanczos_steps must be >= 2");
  if (c.trace_probes < 1) fail(ADP_ERR_CONFIG, "solve: trace_probes must be >= 1");
  if (c.p_override < 0) fail(ADP_ERR_CONFIG, "solve: p_override must be >= 1");
}

}  // namespace

// estimate_spectrum_bounds (lanczos.cpp:81-111)
void spectrum_bounds(adp_ctx* ctx, const adp_csr* a, int64_t steps, uint64_t seed, double* lo, double* hi,
                     int64_t* spmv_count) {
  if (a->n_rows != a->n_cols) fail(ADP_ERR_DIMENSION, "estimate_spectrum_bounds: matrix not square");
  if (a->n_rows == 0) fail(ADP_ERR_DIMENSION, "estimate_spectrum_bounds: empty matrix");
  if (steps < 2) fail(ADP_ERR_CONFIG, "estimate_spectrum_bounds: need steps >= 2");
  if (a->dtype != ADP_F64) fail(ADP_ERR_CONFIG, "solve: real symmetric operators only (the reference's scope)");
  const int64_t n = a->n_rows;
  const int64_t eff = std::min<int64_t>(steps, n);
  double lower = std::numeric_limits<double>::infinity(), upper = -std::numeric_limits<double>::infinity();
  for (int attempt = 0; attempt <= 3; ++attempt) {
    const LanczosRun run = lanczos_pass(ctx, a, eff, seed, static_cast<uint64_t>(attempt) * n, spmv_count);
    lower = std::min(lower, run.lower);
    upper = std::max(upper, run.upper);
    if (!run.early_breakdown) break;
  }
  const double magnitude = std::max(std::abs(lower), std::abs(upper));
  if (!(upper - lower > 1e-12 * magnitude)) {
    const double pad = std::max(1e-8, std::numeric_limits<double>::epsilon() * static_cast<double>(n) * magnitude);
    lower -= pad;
    upper += pad;
  }
  *lo = lower;
  *hi = upper;
}

// estimate_eigcount (solver.cpp:108-117)
double eigcount(adp_ctx* ctx, const adp_csr* a, const double* coeffs, int k_max, double l1, double l2, int64_t probes,
                uint64_t seed, int64_t* spmv_count) {
  if (probes < 1) fail(ADP_ERR_CONFIG, "estimate_eigcount: need at least one probe");
  const int64_t n = a->n_rows;
  std::vector<double> v(static_cast<size_t>(n) * probes);
  check_status(adp_fill_rademacher(v.data(), n, probes, seed, 2));
  DeviceBlock vd(n, probes), wd(n, probes);
  upload_colmajor(ctx, v.data(), n, probes, vd);
  check_status(adp_filter_apply_device(ctx, a, coeffs, k_max, l1, l2, k_max, vd.ptr, n, vd.ld, probes, wd.ptr, wd.ld,
                                       spmv_count));
  const std::vector<double> dots =
      column_reduce(ctx, vd.ptr, vd.ld, wd.ptr, wd.ld, {}, n, static_cast<int32_t>(probes), 1);
  double acc = 0.0;
  for (double d : dots) acc += d;
  return acc / static_cast<double>(probes);
}

}  // namespace adp

// ================================================================== solve ===
struct adp_solve_result {
  adp_solve_summary summary{};
  std::vector<double> eigenvalues;
  std::vector<double> eigenvectors;  // column-major n x e
  std::vector<adp_iteration_record> history;
  std::vector<int32_t> degree_history;
};

namespace adp {
namespace {

// top_up_basis (solver.cpp:58-77) on a device block whose first `have` columns
// are orthonormal; fills columns have..target-1.
void top_up(adp_ctx* ctx, DeviceBlock& q, int64_t n, int64_t have, int64_t target, uint64_t seed,
            uint64_t draw_offset) {
  DeviceVec v(n), h(std::max<int64_t>(target, 1));
  std::vector<double> hv(n);
  uint64_t draw = draw_offset;
  while (have < target) {
    check_status(adp_philox_gaussian(seed, 3, draw, n, hv.data()));
    draw += static_cast<uint64_t>(n);
    ADP_CUDA(cudaMemcpyAsync(v.ptr, hv.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
    for (int pass = 0; pass < 2 && have > 0; ++pass) {
      // row-major n x have block == column-major have x n matrix M: Q^T v = M v, Q h = M^T h
      gemv(ctx, false, have, n, 1.0, q.ptr, q.ld, v.ptr, 1, 0.0, h.ptr, 1);
      gemv(ctx, true, have, n, -1.0, q.ptr, q.ld, h.ptr, 1, 1.0, v.ptr, 1);
    }
    const double nrm = nrm2(ctx, v.ptr, n, 1);
    sync(ctx);
    if (nrm <= 1e-8) continue;
    scal(ctx, 1.0 / nrm, v.ptr, 1, n);
    ADP_CUDA(cudaMemcpy2DAsync(q.ptr + have, q.ld * 8, v.ptr, 8, 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
    ++have;
  }
  sync(ctx);
}

// ||[L A]^T [L A] - I||_F for the joint basis (diagnostics, solver.cpp:244-250)
double orth_error(adp_ctx* ctx, const DeviceBlock& joint, int64_t n, int64_t p) {
  std::vector<double> g(static_cast<size_t>(p) * p);
  DeviceVec gd(p * p);
  // G = M M^T with M = joint^T (p x n, ld)
  for (int64_t j = 0; j < p; ++j)
    gemv(ctx, false, p, n, 1.0, joint.ptr, joint.ld, joint.ptr + j, joint.ld, 0.0, gd.ptr + j * p, 1);
  ADP_CUDA(cudaMemcpyAsync(g.data(), gd.ptr, static_cast<size_t>(p) * p * 8, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  double s = 0.0;
  for (int64_t j = 0; j < p; ++j)
    for (int64_t i = 0; i < p; ++i) {
      const double d = g[i + j * p] - (i == j ? 1.0 : 0.0);
      s += d * d;
    }
  return std::sqrt(s);
}

void emit_pairs(adp_ctx* ctx, adp_solve_result& res, const std::vector<double>& values, const double* vecs, int64_t ld,
                int64_t n, int64_t count, DeviceBlock& scratch) {
  std::vector<int32_t> order(count);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t i, int32_t j) { return values[i] < values[j]; });
  res.eigenvalues.resize(count);
  for (int64_t i = 0; i < count; ++i) res.eigenvalues[i] = values[order[i]];
  res.eigenvectors.assign(static_cast<size_t>(n) * count, 0.0);
  if (count == 0) return;
  gather_columns(ctx, vecs, ld, n, order, scratch.ptr, scratch.ld);
  download_colmajor(ctx, scratch.ptr, scratch.ld, n, count, res.eigenvectors.data());
}

}  // namespace

adp_solve_result* solve(adp_ctx* ctx, const adp_csr* a, const adp_solver_config& cfg) {
  validate_config(cfg);
  if (a->n_rows != a->n_cols) fail(ADP_ERR_DIMENSION, "solve: matrix not square");
  auto res = std::make_unique<adp_solve_result>();
  adp_solve_summary& S = res->summary;
  const int64_t n = a->n_rows;
  S.n = n;
  const double lo = cfg.interval_a, hi = cfg.interval_b;
  const auto setup_start = Clock::now();

  // --- setup: spectrum bounds, filter, eigenvalue count, subspace size (solver.cpp:129-176)
  spectrum_bounds(ctx, a, cfg.lanczos_steps, cfg.rng_seed, &S.lambda_min, &S.lambda_max, &S.spmv_total);
  if (!(S.lambda_min <= lo && hi <= S.lambda_max))
    fail(ADP_ERR_CONFIG, "solve: target interval lies outside the estimated spectrum [" +
                             std::to_string(S.lambda_min) + ", " + std::to_string(S.lambda_max) + "]");
  const double a_norm = std::max(std::abs(S.lambda_min), std::abs(S.lambda_max));
  const double span = S.lambda_max - S.lambda_min;
  const double l1 = 2.0 / span, l2 = -(S.lambda_max + S.lambda_min) / span;
  auto mapc = [&](double x) { return std::clamp(l1 * x + l2, -1.0, 1.0); };
  const double alpha = std::acos(mapc(lo)), beta = std::acos(mapc(hi));
  if (!(alpha > beta)) fail(ADP_ERR_CONFIG, "solve: interval collapses under the spectral map");
  int32_t k1 = 0;
  check_status(adp_initial_degree(alpha, beta, cfg.c, &k1));
  const int32_t k_max = std::max<int32_t>(k1, static_cast<int32_t>(std::ceil(cfg.k_multiplier * static_cast<double>(k1))));
  adp_filter_info f{};
  std::vector<double> coeffs(static_cast<size_t>(k_max) + 1);
  check_status(adp_build_filter(lo, hi, S.lambda_min, S.lambda_max, k_max, cfg.m, ADP_DAMP_LANCZOS, &f, coeffs.data()));

  S.e_estimate = eigcount(ctx, a, coeffs.data(), k_max, f.l1, f.l2, cfg.trace_probes, cfg.rng_seed, &S.spmv_total);

  int64_t p = 0;
  if (cfg.p_override > 0) {
    p = cfg.p_override;
  } else {
    if (S.e_estimate < 0.5) {
      S.converged = 1;
      S.timings.setup = seconds_since(setup_start);
      return res.release();
    }
    const int64_t e_ceil = static_cast<int64_t>(std::ceil(std::max(S.e_estimate, 0.0)));
    p = std::max<int64_t>({static_cast<int64_t>(std::ceil(cfg.mu * static_cast<double>(e_ceil))), e_ceil + 5, 10});
  }
  S.subspace_dim = std::min(p, n);

  if (p >= n) {  // dense fallback (solver.cpp:178-198)
    std::vector<double> dense(static_cast<size_t>(n) * n, 0.0);
    ensure_host_copy(const_cast<adp_csr*>(a));
    const double* hv = static_cast<const double*>(a->h_values);
    for (int64_t r = 0; r < n; ++r)
      for (int64_t k = a->h_row_ptr[r]; k < a->h_row_ptr[r + 1]; ++k) dense[r + static_cast<size_t>(a->h_col[k]) * n] += hv[k];
    DeviceVec dd(n * n);
    ADP_CUDA(cudaMemcpyAsync(dd.ptr, dense.data(), dense.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    const std::vector<double> ev = sym_eig_device(ctx, dd.ptr, static_cast<int32_t>(n));
    // eigenvectors: column-major n x n (column i pairs with ev[i]) == row-major block whose ROW i is vector i
    std::vector<int32_t> sel;
    std::vector<double> vals;
    for (int64_t i = 0; i < n; ++i)
      if (ev[i] >= lo && ev[i] <= hi) {
        sel.push_back(static_cast<int32_t>(i));
        vals.push_back(ev[i]);
      }
    DeviceBlock vecs(n, std::max<int64_t>(1, static_cast<int64_t>(sel.size())));
    // transpose the column-major eigenvector matrix into a row-major n x n block, then gather
    DeviceBlock full(n, n);
    launch_colmajor_to_rowmajor(ctx, dd.ptr, n, n, n, full.ptr, full.ld, 8);
    gather_columns(ctx, full.ptr, full.ld, n, sel, vecs.ptr, vecs.ld);
    DeviceBlock scratch(n, std::max<int64_t>(1, static_cast<int64_t>(sel.size())));
    emit_pairs(ctx, *res, vals, vecs.ptr, vecs.ld, n, static_cast<int64_t>(sel.size()), scratch);
    S.n_eigs = static_cast<int64_t>(res->eigenvalues.size());
    if (S.n_eigs > 0) {
      DeviceBlock ev_blk(n, S.n_eigs), av(n, S.n_eigs);
      upload_colmajor(ctx, res->eigenvectors.data(), n, S.n_eigs, ev_blk);
      const std::vector<double> r =
          residual_norms(ctx, a, ev_blk.ptr, ev_blk.ld, static_cast<int32_t>(S.n_eigs), res->eigenvalues, av.ptr);
      S.spmv_total += S.n_eigs;
      S.max_residual = *std::max_element(r.begin(), r.end());
    }
    S.converged = 1;
    S.dense_fallback = 1;
    S.timings.setup = seconds_since(setup_start);
    return res.release();
  }

  // device-resident blocks, all n x p row-major
  DeviceBlock locked(n, p), active(n, p), filtered(n, p), stacked(n, p), scratch(n, p), scratch2(n, p);
  {
    std::vector<double> init(static_cast<size_t>(n) * p);
    check_status(adp_fill_gaussian(init.data(), n, p, cfg.rng_seed, 0));
    upload_colmajor(ctx, init.data(), n, p, active);
  }
  int64_t kept = cholesky_qr(ctx, active.ptr, n, static_cast<int32_t>(p), active.ld);
  if (kept < p) top_up(ctx, active, n, kept, p, cfg.rng_seed, 0);
  int32_t degree = std::min(k1, k_max);
  int64_t n_lock = 0, n_check_prev = 0, iteration = 0;
  std::vector<double> locked_values, ritz;
  S.timings.setup = seconds_since(setup_start);

  int empty_streak = 0;
  while (iteration < cfg.max_iter) {
    ++iteration;
    adp_iteration_record rec{};
    rec.iteration = iteration;
    rec.degree = degree;
    rec.active_width = p - n_lock;
    rec.orth_error = -1.0;
    const int64_t qa = p - n_lock;

    auto t = Clock::now();
    check_status(adp_filter_apply_device(ctx, a, coeffs.data(), k_max, f.l1, f.l2, degree, active.ptr, n, active.ld,
                                         qa, filtered.ptr, filtered.ld, &rec.spmv_filter));
    sync(ctx);
    S.timings.filter += seconds_since(t);

    t = Clock::now();
    copy_columns(ctx, locked.ptr, locked.ld, stacked.ptr, stacked.ld, n, n_lock);
    copy_columns(ctx, filtered.ptr, filtered.ld, stacked.ptr + n_lock, stacked.ld, n, qa);
    kept = cholesky_qr(ctx, stacked.ptr, n, static_cast<int32_t>(p), stacked.ld);
    if (kept < p) top_up(ctx, stacked, n, kept, p, cfg.rng_seed, static_cast<uint64_t>(iteration) << 32);
    sync(ctx);
    S.timings.orth += seconds_since(t);

    t = Clock::now();
    ritz = rayleigh_ritz(ctx, a, stacked.ptr + n_lock, stacked.ld, static_cast<int32_t>(qa), scratch.ptr, active.ptr,
                         active.ld);
    sync(ctx);
    S.timings.rayleigh_ritz += seconds_since(t);

    t = Clock::now();
    if (cfg.collect_diagnostics) {
      copy_columns(ctx, locked.ptr, locked.ld, scratch.ptr, scratch.ld, n, n_lock);
      copy_columns(ctx, active.ptr, active.ld, scratch.ptr + n_lock, scratch.ld, n, qa);
      rec.orth_error = orth_error(ctx, scratch, n, p);
    }
    std::vector<int32_t> in_interval;
    for (int64_t j = 0; j < qa; ++j)
      if (ritz[j] >= lo && ritz[j] <= hi) in_interval.push_back(static_cast<int32_t>(j));
    const int64_t e_i = static_cast<int64_t>(in_interval.size());
    rec.e_in_interval = e_i;
    rec.n_locked_total = n_lock;

    if (e_i == 0) {
      ++empty_streak;
      res->degree_history.push_back(degree);
      res->history.push_back(rec);
      S.iterations = iteration;
      S.timings.other += seconds_since(t);
      if (iteration > 3 && empty_streak >= 10) {
        S.converged = 1;
        break;
      }
      continue;
    }
    empty_streak = 0;
    int32_t next_degree = 0;
    check_status(adp_adaptive_degree(&f, coeffs.data(), ritz.data(), qa, e_i, cfg.tau_a, &next_degree));
    S.timings.other += seconds_since(t);

    t = Clock::now();
    std::vector<double> values_in(e_i);
    for (int64_t c = 0; c < e_i; ++c) values_in[c] = ritz[in_interval[c]];
    gather_columns(ctx, active.ptr, active.ld, n, in_interval, scratch.ptr, scratch.ld);
    const std::vector<double> resid =
        residual_norms(ctx, a, scratch.ptr, scratch.ld, static_cast<int32_t>(e_i), values_in, scratch2.ptr);
    rec.spmv_residual += e_i;
    rec.max_residual = *std::max_element(resid.begin(), resid.end());
    S.timings.residuals += seconds_since(t);

    t = Clock::now();
    double tau_s = std::numeric_limits<double>::infinity();  // spurious_threshold (solver.cpp:81-92)
    for (double x : values_in) tau_s = std::min(tau_s, std::min(x - lo, hi - x));
    std::vector<int64_t> test_set(e_i);
    std::iota(test_set.begin(), test_set.end(), 0);
    if (cfg.spurious_detection && tau_s > 0.0) {
      std::vector<int64_t> checked;
      for (int64_t c = 0; c < e_i; ++c)
        if (resid[c] < tau_s) checked.push_back(c);
      const int64_t n_check = static_cast<int64_t>(checked.size()) + n_lock;
      if (n_check > 0 && n_check == n_check_prev) test_set = checked;
      n_check_prev = n_check;
    }
    const double lock_threshold = cfg.tau_c * a_norm;
    std::vector<char> lock_flag(qa, 0);
    std::vector<int32_t> lock_cols;
    int64_t n_unconverged = 0;
    for (const int64_t c : test_set) {
      if (resid[c] < lock_threshold) {
        const int32_t j = in_interval[c];
        lock_flag[j] = 1;
        locked_values.push_back(ritz[j]);
        lock_cols.push_back(j);
      } else {
        ++n_unconverged;
      }
    }
    const int64_t n_new = static_cast<int64_t>(lock_cols.size());
    if (n_new > 0) {
      gather_columns(ctx, active.ptr, active.ld, n, lock_cols, locked.ptr + n_lock, locked.ld);
      std::vector<int32_t> keep;
      for (int64_t j = 0; j < qa; ++j)
        if (!lock_flag[j]) keep.push_back(static_cast<int32_t>(j));
      gather_columns(ctx, active.ptr, active.ld, n, keep, scratch.ptr, scratch.ld);
      std::swap(active, scratch);
    }
    n_lock += n_new;
    rec.n_locked_total = n_lock;
    res->degree_history.push_back(degree);
    res->history.push_back(rec);
    S.iterations = iteration;
    degree = next_degree;
    S.timings.other += seconds_since(t);
    if (n_unconverged == 0) {
      S.converged = 1;
      break;
    }
  }

  // --- assemble: ascending pairs, re-measured residuals (solver.cpp:346-359)
  emit_pairs(ctx, *res, locked_values, locked.ptr, locked.ld, n, n_lock, scratch);
  S.n_eigs = n_lock;
  if (n_lock > 0) {
    upload_colmajor(ctx, res->eigenvectors.data(), n, n_lock, scratch);
    const std::vector<double> r =
        residual_norms(ctx, a, scratch.ptr, scratch.ld, static_cast<int32_t>(n_lock), res->eigenvalues, scratch2.ptr);
    S.spmv_total += n_lock;
    S.max_residual = *std::max_element(r.begin(), r.end());
  }
  for (const auto& r : res->history) S.spmv_total += r.spmv_filter + r.spmv_residual;
  if (!res->degree_history.empty()) {
    double sd = 0.0;
    for (int32_t d : res->degree_history) sd += d;
    S.avg_degree = sd / static_cast<double>(res->degree_history.size());
  }
  S.n_history = static_cast<int64_t>(res->history.size());
  return res.release();
}

}  // namespace adp

// ==================================================================== C-ABI ===
namespace {
template <class F>
adp_status guarded(F&& f) {
  try {
    f();
    return ADP_OK;
  } catch (const adp::Error& e) {
    adp::set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc& e) {
    adp::set_last_error(std::string("host allocation failed: ") + e.what());
    return ADP_ERR_OOM;
  } catch (const std::exception& e) {
    adp::set_last_error(e.what());
    return ADP_ERR_RUNTIME;
  }
}
}  // namespace

extern "C" {

void adp_solver_config_default(adp_solver_config* c) {  // SolverConfig defaults (solver.hpp:17-31)
  std::memset(c, 0, sizeof(*c));
  c->tau_c = 1e-10;
  c->tau_a = 1e-3;
  c->m = 0.5;
  c->c = 1.4;
  c->k_multiplier = 2.5;
  c->mu = 1.8;
  c->max_iter = 100;
  c->lanczos_steps = 40;
  c->trace_probes = 30;
  c->rng_seed = 0;
  c->p_override = 0;
  c->spurious_detection = 1;
  c->collect_diagnostics = 0;
}

adp_status adp_solve(adp_ctx* ctx, const adp_csr* a, const adp_solver_config* cfg, adp_solve_result** out) {
  return guarded([&] {
    ADP_CUDA(cudaSetDevice(ctx->device));
    *out = adp::solve(ctx, a, *cfg);
  });
}

adp_status adp_solve_summary_get(const adp_solve_result* r, adp_solve_summary* s) {
  return guarded([&] { *s = r->summary; });
}

adp_status adp_solve_eigenpairs(const adp_solve_result* r, double* values, double* vectors, int64_t ldv) {
  return guarded([&] {
    const int64_t e = r->summary.n_eigs, n = r->summary.n;
    if (values) std::copy(r->eigenvalues.begin(), r->eigenvalues.end(), values);
    if (vectors) {
      if (ldv < n) adp::fail(ADP_ERR_DIMENSION, "adp_solve_eigenpairs: ldv < n");
      for (int64_t c = 0; c < e; ++c)
        std::copy(r->eigenvectors.begin() + c * n, r->eigenvectors.begin() + (c + 1) * n, vectors + c * ldv);
    }
  });
}

adp_status adp_solve_history(const adp_solve_result* r, adp_iteration_record* recs, int32_t* degree_history) {
  return guarded([&] {
    if (recs) std::copy(r->history.begin(), r->history.end(), recs);
    if (degree_history) std::copy(r->degree_history.begin(), r->degree_history.end(), degree_history);
  });
}

adp_status adp_solve_result_destroy(adp_solve_result* r) {
  return guarded([&] { delete r; });
}

adp_status adp_spmv_device(adp_ctx* ctx, const adp_csr* a, const double* x, double* y) {
  return guarded([&] {
    ADP_CUDA(cudaSetDevice(ctx->device));
    adp::spmv(ctx, a, x, y);
    ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adp_status adp_lanczos_bounds(adp_ctx* ctx, const adp_csr* a, int32_t steps, uint64_t seed, double* lambda_min,
                              double* lambda_max, int64_t* spmv_count) {
  return guarded([&] { adp::spectrum_bounds(ctx, a, steps, seed, lambda_min, lambda_max, spmv_count); });
}

adp_status adp_estimate_eigcount(adp_ctx* ctx, const adp_csr* a, const double* coeffs, int32_t k_max, double l1,
                                 double l2, int64_t probes, uint64_t seed, double* out, int64_t* spmv_count) {
  return guarded([&] { *out = adp::eigcount(ctx, a, coeffs, k_max, l1, l2, probes, seed, spmv_count); });
}

adp_status adp_cholesky_qr_device(adp_ctx* ctx, double* x, int64_t n, int64_t p, int64_t ld, int64_t* kept) {
  return guarded([&] {
    if (ld < p) adp::fail(ADP_ERR_DIMENSION, "cholesky_qr: ld < p");
    *kept = adp::cholesky_qr(ctx, x, n, static_cast<int32_t>(p), ld);
    ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adp_status adp_rayleigh_ritz_device(adp_ctx* ctx, const adp_csr* a, const double* q, int64_t ld, int64_t qc,
                                    double* theta, double* v_out, int64_t ldv) {
  return guarded([&] {
    if (a->n_rows != a->n_cols) adp::fail(ADP_ERR_DIMENSION, "rayleigh_ritz: basis row count does not match A");
    adp::DeviceBlock aq(a->n_rows, ld);  // own scratch: the spmm workspaces may be re-sized inside
    const std::vector<double> t = adp::rayleigh_ritz(ctx, a, q, ld, static_cast<int32_t>(qc), aq.ptr, v_out, ldv);
    std::copy(t.begin(), t.end(), theta);
  });
}

adp_status adp_residual_norms_device(adp_ctx* ctx, const adp_csr* a, const double* v, int64_t ld, int64_t e,
                                     const double* lam, double* norms) {
  return guarded([&] {
    std::vector<double> l(lam, lam + e);
    adp::DeviceBlock av(a->n_rows, ld);
    const std::vector<double> r = adp::residual_norms(ctx, a, v, ld, static_cast<int32_t>(e), l, av.ptr);
    std::copy(r.begin(), r.end(), norms);
  });
}

adp_status adp_spurious_threshold(const double* ritz, int64_t n, double a, double b, double* out) {
  return guarded([&] {  // solver.cpp:81-92
    if (n == 0) adp::fail(ADP_ERR_CONFIG, "spurious_threshold: empty Ritz set");
    double tau = std::numeric_limits<double>::infinity();
    for (int64_t i = 0; i < n; ++i) {
      const double x = ritz[i];
      if (x < a || x > b) adp::fail(ADP_ERR_CONFIG, "spurious_threshold: Ritz value outside the interval");
      tau = std::min(tau, std::min(x - a, b - x));
    }
    *out = tau;
  });
}

}  // extern "C"
