// Dense device subsystems of the solver: CholQR2 with the reference's fallback
// chain, Rayleigh-Ritz, residual norms, column gathers and reductions.
//
// Blocks are row-major n x p with leading dimension ld (the kernel layout). To
// cuBLAS / cuSOLVER (column-major) such a block is M = X^T, a p x n matrix with
// leading dimension ld, so:
//   Gram      G = X^T X        = M M^T           (syrk, upper)
//   X R^{-1}  (X R^{-1})^T     = R^{-T} M        (trsm left, upper, transposed)
//   B = Q^T A Q                = M_Q M_AQ^T      (gemm N,T)
//   V = Q U   (Q U)^T          = U^T M_Q         (gemm T,N)
// Mirrors proj/src/dense_kernels.cpp (cholesky :41-51, cholesky_qr :53-92,
// mgs_orthonormalize :12-27, rayleigh_ritz :94-101, sym_eig :31-39) and
// compute_residuals (proj/src/solver.cpp:94-106).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "adp_internal.hpp"
#include "dense.hpp"

namespace adp {

namespace {

#define ADP_CUBLAS(call)                                                                   \
  do {                                                                                     \
    cublasStatus_t st__ = (call);                                                          \
    if (st__ != CUBLAS_STATUS_SUCCESS)                                                     \
      ::adp::fail(ADP_ERR_CUDA, std::string(#call) + ": cublas status " + std::to_string(st__)); \
  } while (0)
#define ADP_CUSOLVER(call)                                                                   \
  do {                                                                                       \
    cusolverStatus_t st__ = (call);                                                          \
    if (st__ != CUSOLVER_STATUS_SUCCESS)                                                     \
      ::adp::fail(ADP_ERR_CUDA, std::string(#call) + ": cusolver status " + std::to_string(st__)); \
  } while (0)

struct Handles {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t sol = nullptr;
  int* d_info = nullptr;
  DevBuf work, g, g2, diag, part, idx, tmp, evals;
};

Handles& handles(adp_ctx* ctx) {
  if (!ctx->cublas) {
    auto* h = new Handles;
    ADP_CUDA(cudaSetDevice(ctx->device));
    ADP_CUBLAS(cublasCreate(&h->blas));
    ADP_CUSOLVER(cusolverDnCreate(&h->sol));
    ADP_CUDA(cudaMalloc(&h->d_info, sizeof(int)));
    ctx->cublas = h;
  }
  auto* h = static_cast<Handles*>(ctx->cublas);
  ADP_CUBLAS(cublasSetStream(h->blas, ctx->stream));
  ADP_CUSOLVER(cusolverDnSetStream(h->sol, ctx->stream));
  return *h;
}

// ---- kernels ------------------------------------------------------------------------
__global__ void gather_cols_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                                   int64_t ldd, int64_t n, const int32_t* __restrict__ idx, int32_t m) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * m;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / m;
    const int32_t j = static_cast<int32_t>(t - r * m);
    dst[r * ldd + j] = src[r * lds + idx[j]];
  }
}

// Per-column partial reductions over row chunks, then a fixed-order final sum:
// deterministic for a fixed launch geometry.
//   kind 0: sum_r (a[r][j] - lam_j b[r][j])^2      (residual norms^2)
//   kind 1: sum_r a[r][j] * b[r][j]                  (column dots)
constexpr int kRedRows = 1024;
__global__ void col_partials_kernel(const double* __restrict__ a, int64_t lda, const double* __restrict__ b,
                                    int64_t ldb, const double* __restrict__ lam, int64_t n, int32_t m, int kind,
                                    double* __restrict__ part) {
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRedRows;
  const int64_t r1 = min(n, r0 + kRedRows);
  for (int32_t j = threadIdx.x; j < m; j += blockDim.x) {
    double acc = 0.0;
    const double l = kind == 0 ? lam[j] : 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      const double x = a[r * lda + j];
      const double y = b[r * ldb + j];
      if (kind == 0) {
        const double d = __dsub_rn(x, __dmul_rn(l, y));
        acc = __dadd_rn(acc, __dmul_rn(d, d));
      } else {
        acc = __dadd_rn(acc, __dmul_rn(x, y));
      }
    }
    part[static_cast<int64_t>(blockIdx.x) * m + j] = acc;
  }
}
__global__ void col_final_kernel(const double* __restrict__ part, int64_t nblocks, int32_t m, double* __restrict__ out) {
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t b = 0; b < nblocks; ++b) acc = __dadd_rn(acc, part[b * m + j]);
    out[j] = acc;
  }
}

// y = A x, one thread per row, sequential accumulation in CSR order: the
// reference's csr_spmv (proj/include/adapoly/csr_matrix.hpp:122-134).
template <class RP>
__global__ void spmv_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
                            const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (RP k = rp[r]; k < rp[r + 1]; ++k) acc = __dadd_rn(acc, __dmul_rn(val[k], x[col[k]]));
    y[r] = acc;
  }
}

__global__ void symmetrize_kernel(double* b, int32_t p) {  // (B + B^T) / 2, column-major p x p
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < int64_t{p} * p;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = static_cast<int32_t>(t % p), j = static_cast<int32_t>(t / p);
    if (i < j) {
      const double s = __dmul_rn(0.5, __dadd_rn(b[i + int64_t{j} * p], b[j + int64_t{i} * p]));
      b[i + int64_t{j} * p] = s;
      b[j + int64_t{i} * p] = s;
    }
  }
}

__global__ void add_diag_kernel(double* g, int32_t p, double shift) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p) g[i + int64_t{i} * p] = __dadd_rn(g[i + int64_t{i} * p], shift);
}

__global__ void copy_diag_kernel(const double* g, int32_t p, double* d) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p) d[i] = g[i + int64_t{i} * p];
}

__global__ void fill_lower_from_upper_kernel(double* g, int32_t p) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < int64_t{p} * p;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t i = static_cast<int32_t>(t % p), j = static_cast<int32_t>(t / p);
    if (i > j) g[i + int64_t{j} * p] = g[j + int64_t{i} * p];
  }
}

int blocks_for(int64_t work, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads, 148 * 16)));
}

}  // namespace

void release_dense(adp_ctx* ctx) {
  if (!ctx->cublas) return;
  auto* h = static_cast<Handles*>(ctx->cublas);
  cublasDestroy(h->blas);
  cusolverDnDestroy(h->sol);
  cudaFree(h->d_info);
  h->work.release();
  h->g.release();
  h->g2.release();
  h->diag.release();
  h->part.release();
  h->idx.release();
  h->tmp.release();
  h->evals.release();
  delete h;
  ctx->cublas = nullptr;
}

// ---- column operations ------------------------------------------------------------------
void gather_columns(adp_ctx* ctx, const double* src, int64_t lds, int64_t n, const std::vector<int32_t>& cols,
                    double* dst, int64_t ldd) {
  if (cols.empty() || n == 0) return;
  Handles& h = handles(ctx);
  auto* d_idx = static_cast<int32_t*>(h.idx.get(cols.size() * sizeof(int32_t)));
  ADP_CUDA(cudaMemcpyAsync(d_idx, cols.data(), cols.size() * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
  const int32_t m = static_cast<int32_t>(cols.size());
  gather_cols_kernel<<<blocks_for(n * m), 256, 0, ctx->stream>>>(src, lds, dst, ldd, n, d_idx, m);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
  // the index buffer is reused by the next call: keep the host vector alive until the copy is done
  ADP_CUDA(cudaStreamSynchronize(ctx->stream));
}

void copy_columns(adp_ctx* ctx, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t n, int64_t m) {
  if (n == 0 || m == 0) return;
  ADP_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, src, lds * 8, m * 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
}

std::vector<double> column_reduce(adp_ctx* ctx, const double* a, int64_t lda, const double* b, int64_t ldb,
                                  const std::vector<double>& lam, int64_t n, int32_t m, int kind) {
  std::vector<double> out(m, 0.0);
  if (m == 0) return out;
  Handles& h = handles(ctx);
  const int64_t nb = std::max<int64_t>(1, (n + kRedRows - 1) / kRedRows);
  auto* part = static_cast<double*>(h.part.get(static_cast<size_t>(nb) * m * 8 + m * 8 + m * 8));
  double* d_lam = part + nb * m;
  double* d_out = d_lam + m;
  if (kind == 0)
    ADP_CUDA(cudaMemcpyAsync(d_lam, lam.data(), m * 8, cudaMemcpyHostToDevice, ctx->stream));
  col_partials_kernel<<<static_cast<unsigned>(nb), 256, 0, ctx->stream>>>(a, lda, b, ldb, d_lam, n, m, kind, part);
  ADP_LAUNCH_CHECK();
  col_final_kernel<<<blocks_for(m), 256, 0, ctx->stream>>>(part, nb, m, d_out);
  ADP_LAUNCH_CHECK();
  ctx->launches += 2;
  ADP_CUDA(cudaMemcpyAsync(out.data(), d_out, m * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  return out;
}

void spmv(adp_ctx* ctx, const adp_csr* a, const double* x, double* y) {
  if (a->dtype != ADP_F64) fail(ADP_ERR_CONFIG, "spmv: real operators only");
  const int grid = blocks_for(a->n_rows);
  if (a->rp64)
    spmv_kernel<int64_t><<<grid, 256, 0, ctx->stream>>>(static_cast<const int64_t*>(a->row_ptr), a->col_idx,
                                                        static_cast<const double*>(a->values), x, y, a->n_rows);
  else
    spmv_kernel<int32_t><<<grid, 256, 0, ctx->stream>>>(static_cast<const int32_t*>(a->row_ptr), a->col_idx,
                                                        static_cast<const double*>(a->values), x, y, a->n_rows);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

double dot(adp_ctx* ctx, const double* x, const double* y, int64_t n, int64_t incx, int64_t incy) {
  Handles& h = handles(ctx);
  double r = 0.0;
  ADP_CUBLAS(cublasSetPointerMode(h.blas, CUBLAS_POINTER_MODE_HOST));
  ADP_CUBLAS(cublasDdot(h.blas, static_cast<int>(n), x, static_cast<int>(incx), y, static_cast<int>(incy), &r));
  return r;
}

double nrm2(adp_ctx* ctx, const double* x, int64_t n, int64_t incx) {
  Handles& h = handles(ctx);
  double r = 0.0;
  ADP_CUBLAS(cublasSetPointerMode(h.blas, CUBLAS_POINTER_MODE_HOST));
  ADP_CUBLAS(cublasDnrm2(h.blas, static_cast<int>(n), x, static_cast<int>(incx), &r));
  return r;
}

void axpy(adp_ctx* ctx, double alpha, const double* x, int64_t incx, double* y, int64_t incy, int64_t n) {
  Handles& h = handles(ctx);
  ADP_CUBLAS(cublasSetPointerMode(h.blas, CUBLAS_POINTER_MODE_HOST));
  ADP_CUBLAS(cublasDaxpy(h.blas, static_cast<int>(n), &alpha, x, static_cast<int>(incx), y, static_cast<int>(incy)));
}

void scal(adp_ctx* ctx, double alpha, double* x, int64_t incx, int64_t n) {
  Handles& h = handles(ctx);
  ADP_CUBLAS(cublasSetPointerMode(h.blas, CUBLAS_POINTER_MODE_HOST));
  ADP_CUBLAS(cublasDscal(h.blas, static_cast<int>(n), &alpha, x, static_cast<int>(incx)));
}

// y = alpha op(A) x + beta y with A column-major (m x k, lda)
void gemv(adp_ctx* ctx, bool trans, int64_t m, int64_t k, double alpha, const double* a, int64_t lda, const double* x,
          int64_t incx, double beta, double* y, int64_t incy) {
  Handles& h = handles(ctx);
  ADP_CUBLAS(cublasSetPointerMode(h.blas, CUBLAS_POINTER_MODE_HOST));
  ADP_CUBLAS(cublasDgemv(h.blas, trans ? CUBLAS_OP_T : CUBLAS_OP_N, static_cast<int>(m), static_cast<int>(k), &alpha,
                         a, static_cast<int>(lda), x, static_cast<int>(incx), &beta, y, static_cast<int>(incy)));
}

// ---- CholQR2 ------------------------------------------------------------------------------
namespace {

// G = X^T X (upper triangle, column-major p x p) for a row-major n x p block.
void gram_upper(adp_ctx* ctx, const double* x, int64_t n, int32_t p, int64_t ld, double* g) {
  Handles& h = handles(ctx);
  const double one = 1.0, zero = 0.0;
  ADP_CUBLAS(cublasSetPointerMode(h.blas, CUBLAS_POINTER_MODE_HOST));
  ADP_CUBLAS(cublasDsyrk(h.blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, p, static_cast<int>(n), &one, x,
                         static_cast<int>(ld), &zero, g, p));
}

// In-place upper Cholesky G = R^T R; false on a non-positive pivot (NotPositiveDefinite).
bool potrf_upper(adp_ctx* ctx, double* g, int32_t p) {
  Handles& h = handles(ctx);
  int lwork = 0;
  ADP_CUSOLVER(cusolverDnDpotrf_bufferSize(h.sol, CUBLAS_FILL_MODE_UPPER, p, g, p, &lwork));
  auto* work = static_cast<double*>(h.work.get(static_cast<size_t>(std::max(lwork, 1)) * 8));
  ADP_CUSOLVER(cusolverDnDpotrf(h.sol, CUBLAS_FILL_MODE_UPPER, p, g, p, work, lwork, h.d_info));
  int info = 0;
  ADP_CUDA(cudaMemcpyAsync(&info, h.d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (info != 0) return false;
  // cholesky() also rejects non-finite factors and non-positive diagonals (dense_kernels.cpp:46-50)
  std::vector<double> d(p);
  auto* dd = static_cast<double*>(h.diag.get(static_cast<size_t>(p) * 8));
  copy_diag_kernel<<<(p + 255) / 256, 256, 0, ctx->stream>>>(g, p, dd);
  ADP_LAUNCH_CHECK();
  ADP_CUDA(cudaMemcpyAsync(d.data(), dd, p * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  for (double v : d)
    if (!std::isfinite(v) || !(v > 0.0)) return false;
  return true;
}

std::vector<double> diag_host(adp_ctx* ctx, const double* g, int32_t p) {
  Handles& h = handles(ctx);
  std::vector<double> d(p);
  auto* dd = static_cast<double*>(h.diag.get(static_cast<size_t>(p) * 8));
  copy_diag_kernel<<<(p + 255) / 256, 256, 0, ctx->stream>>>(g, p, dd);
  ADP_LAUNCH_CHECK();
  ADP_CUDA(cudaMemcpyAsync(d.data(), dd, p * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  return d;
}

// X <- X R^{-1}
void trsm_right_upper(adp_ctx* ctx, const double* r, int32_t p, double* x, int64_t n, int64_t ld) {
  Handles& h = handles(ctx);
  const double one = 1.0;
  ADP_CUBLAS(cublasSetPointerMode(h.blas, CUBLAS_POINTER_MODE_HOST));
  ADP_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, p,
                         static_cast<int>(n), &one, r, p, x, static_cast<int>(ld)));
}

}  // namespace

// mgs_orthonormalize (dense_kernels.cpp:12-27): modified Gram-Schmidt with one
// re-orthogonalisation pass; columns collapsing below 1e-13 of their norm are
// dropped. Kept columns are compacted to the left; returns their count.
int32_t mgs_orthonormalize(adp_ctx* ctx, double* x, int64_t n, int32_t p, int64_t ld) {
  Handles& h = handles(ctx);
  auto* v = static_cast<double*>(h.tmp.get(static_cast<size_t>(n) * 8));
  int32_t kept = 0;
  for (int32_t j = 0; j < p; ++j) {
    ADP_CUBLAS(cublasDcopy(h.blas, static_cast<int>(n), x + j, static_cast<int>(ld), v, 1));
    const double orig = nrm2(ctx, v, n, 1);
    for (int pass = 0; pass < 2; ++pass)
      for (int32_t i = 0; i < kept; ++i) {
        const double c = dot(ctx, x + i, v, n, ld, 1);
        axpy(ctx, -c, x + i, ld, v, 1, n);
      }
    const double nrm = nrm2(ctx, v, n, 1);
    if (!(nrm > orig * 1e-13) || !(nrm > 0.0)) continue;
    scal(ctx, 1.0 / nrm, v, 1, n);
    ADP_CUBLAS(cublasDcopy(h.blas, static_cast<int>(n), v, 1, x + kept, static_cast<int>(ld)));
    ++kept;
  }
  return kept;
}

// cholesky_qr (dense_kernels.cpp:53-92): in place on a row-major n x p block;
// returns the number of orthonormal columns (compacted to the left).
int32_t cholesky_qr(adp_ctx* ctx, double* x, int64_t n, int32_t p, int64_t ld) {
  if (p == 0) return 0;
  Handles& h = handles(ctx);
  auto* g = static_cast<double*>(h.g.get(static_cast<size_t>(p) * p * 8));
  bool first_ok = false;
  {
    gram_upper(ctx, x, n, p, ld, g);
    std::vector<double> gd = diag_host(ctx, g, p);
    for (double v : gd)
      if (!std::isfinite(v)) fail(ADP_ERR_RUNTIME, "cholesky_qr: non-finite entries");
    auto* g2 = static_cast<double*>(h.g2.get(static_cast<size_t>(p) * p * 8));
    ADP_CUDA(cudaMemcpyAsync(g2, g, static_cast<size_t>(p) * p * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    bool ok = potrf_upper(ctx, g2, p);
    if (!ok) {  // shift retry: 1e-14 * trace / p (dense_kernels.cpp:64-68)
      double tr = 0.0;
      for (double v : gd) tr += v;
      const double shift = 1e-14 * tr / static_cast<double>(p);
      add_diag_kernel<<<(p + 255) / 256, 256, 0, ctx->stream>>>(g, p, shift);
      ADP_LAUNCH_CHECK();
      gd = diag_host(ctx, g, p);
      ADP_CUDA(cudaMemcpyAsync(g2, g, static_cast<size_t>(p) * p * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      ok = potrf_upper(ctx, g2, p);
    }
    if (ok) {
      // rank check: r_jj > 1e-7 sqrt(g_jj) (dense_kernels.cpp:73-75)
      const std::vector<double> rd = diag_host(ctx, g2, p);
      for (int32_t j = 0; j < p; ++j)
        if (!(rd[j] > 1e-7 * std::sqrt(gd[j]))) ok = false;
    }
    if (ok) {
      trsm_right_upper(ctx, g2, p, x, n, ld);
      first_ok = true;
    }
  }
  if (!first_ok) return mgs_orthonormalize(ctx, x, n, p, ld);
  // second pass (CholeskyQR2)
  gram_upper(ctx, x, n, p, ld, g);
  if (!potrf_upper(ctx, g, p)) return mgs_orthonormalize(ctx, x, n, p, ld);
  trsm_right_upper(ctx, g, p, x, n, ld);
  return p;
}

// rayleigh_ritz (dense_kernels.cpp:94-101) on a row-major n x q orthonormal
// block Q: V = Q U where (Q^T A Q + (Q^T A Q)^T)/2 = U diag(theta) U^T, theta
// ascending (returned). `aq` is caller scratch of the same shape as Q.
std::vector<double> rayleigh_ritz(adp_ctx* ctx, const adp_csr* a, const double* q, int64_t ld, int32_t qc,
                                  double* aq, double* v_out, int64_t ldv) {
  std::vector<double> theta(qc);
  if (qc == 0) return theta;
  const int64_t n = a->n_rows;
  check_status(adp_spmm_device(ctx, a, q, n, ld, qc, aq, ld, 0));
  Handles& h = handles(ctx);
  auto* b = static_cast<double*>(h.g.get(static_cast<size_t>(qc) * qc * 8));
  const double one = 1.0, zero = 0.0;
  ADP_CUBLAS(cublasSetPointerMode(h.blas, CUBLAS_POINTER_MODE_HOST));
  ADP_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_T, qc, qc, static_cast<int>(n), &one, q, static_cast<int>(ld),
                         aq, static_cast<int>(ld), &zero, b, qc));
  symmetrize_kernel<<<blocks_for(int64_t{qc} * qc), 256, 0, ctx->stream>>>(b, qc);
  ADP_LAUNCH_CHECK();
  auto* w = static_cast<double*>(h.evals.get(static_cast<size_t>(qc) * 8));
  int lwork = 0;
  ADP_CUSOLVER(cusolverDnDsyevd_bufferSize(h.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, qc, b, qc, w,
                                           &lwork));
  auto* work = static_cast<double*>(h.work.get(static_cast<size_t>(std::max(lwork, 1)) * 8));
  ADP_CUSOLVER(cusolverDnDsyevd(h.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, qc, b, qc, w, work, lwork,
                                h.d_info));
  int info = 0;
  ADP_CUDA(cudaMemcpyAsync(&info, h.d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaMemcpyAsync(theta.data(), w, static_cast<size_t>(qc) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (info != 0) fail(ADP_ERR_RUNTIME, "sym_eig: decomposition failed to converge");
  // V^T = U^T Q^T
  ADP_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, qc, static_cast<int>(n), qc, &one, b, qc, q,
                         static_cast<int>(ld), &zero, v_out, static_cast<int>(ldv)));
  return theta;
}

// Dense symmetric eigendecomposition of a small column-major matrix on the
// device (sym_eig, dense_kernels.cpp:31-39): symmetrised, ascending.
std::vector<double> sym_eig_device(adp_ctx* ctx, double* b, int32_t p) {
  Handles& h = handles(ctx);
  std::vector<double> theta(p);
  symmetrize_kernel<<<blocks_for(int64_t{p} * p), 256, 0, ctx->stream>>>(b, p);
  ADP_LAUNCH_CHECK();
  auto* w = static_cast<double*>(h.evals.get(static_cast<size_t>(p) * 8));
  int lwork = 0;
  ADP_CUSOLVER(cusolverDnDsyevd_bufferSize(h.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, p, b, p, w, &lwork));
  auto* work = static_cast<double*>(h.work.get(static_cast<size_t>(std::max(lwork, 1)) * 8));
  ADP_CUSOLVER(cusolverDnDsyevd(h.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, p, b, p, w, work, lwork,
                                h.d_info));
  int info = 0;
  ADP_CUDA(cudaMemcpyAsync(&info, h.d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaMemcpyAsync(theta.data(), w, static_cast<size_t>(p) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (info != 0) fail(ADP_ERR_RUNTIME, "sym_eig: decomposition failed to converge");
  return theta;
}

// compute_residuals (solver.cpp:94-106): ||A v_j - lambda_j v_j||_2 for the
// columns of a row-major n x e block; `av` is caller scratch of the same shape.
std::vector<double> residual_norms(adp_ctx* ctx, const adp_csr* a, const double* v, int64_t ld, int32_t e,
                                   const std::vector<double>& lam, double* av) {
  std::vector<double> r(e);
  if (e == 0) return r;
  check_status(adp_spmm_device(ctx, a, v, a->n_cols, ld, e, av, ld, 0));
  std::vector<double> s = column_reduce(ctx, av, ld, v, ld, lam, a->n_rows, e, 0);
  for (int32_t j = 0; j < e; ++j) r[j] = std::sqrt(s[j]);
  return r;
}

void check_status(adp_status s) {
  if (s != ADP_OK) fail(s, adp_last_error_message());
}

}  // namespace adp

extern "C" void adp_release_dense_handles(adp_ctx* ctx) { adp::release_dense(ctx); }
