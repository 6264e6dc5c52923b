// Device dense helpers shared by the solver translation units (dense.cu).
#pragma once

#include <vector>

#include "adp_internal.hpp"

namespace adp {

void check_status(adp_status s);
void release_dense(adp_ctx* ctx);

// row-major blocks: element (r, c) at base[r * ld + c]
void gather_columns(adp_ctx* ctx, const double* src, int64_t lds, int64_t n, const std::vector<int32_t>& cols,
                    double* dst, int64_t ldd);
void copy_columns(adp_ctx* ctx, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t n, int64_t m);
// kind 0: sum_r (a - lam_j b)^2 ; kind 1: sum_r a * b  (per column, deterministic order)
std::vector<double> column_reduce(adp_ctx* ctx, const double* a, int64_t lda, const double* b, int64_t ldb,
                                  const std::vector<double>& lam, int64_t n, int32_t m, int kind);

// vectors
void spmv(adp_ctx* ctx, const adp_csr* a, const double* x, double* y);
double dot(adp_ctx* ctx, const double* x, const double* y, int64_t n, int64_t incx, int64_t incy);
double nrm2(adp_ctx* ctx, const double* x, int64_t n, int64_t incx);
void axpy(adp_ctx* ctx, double alpha, const double* x, int64_t incx, double* y, int64_t incy, int64_t n);
void scal(adp_ctx* ctx, double alpha, double* x, int64_t incx, int64_t n);
void gemv(adp_ctx* ctx, bool trans, int64_t m, int64_t k, double alpha, const double* a, int64_t lda, const double* x,
          int64_t incx, double beta, double* y, int64_t incy);

// subsystems
int32_t mgs_orthonormalize(adp_ctx* ctx, double* x, int64_t n, int32_t p, int64_t ld);
int32_t cholesky_qr(adp_ctx* ctx, double* x, int64_t n, int32_t p, int64_t ld);
std::vector<double> rayleigh_ritz(adp_ctx* ctx, const adp_csr* a, const double* q, int64_t ld, int32_t qc,
                                  double* aq, double* v_out, int64_t ldv);
std::vector<double> sym_eig_device(adp_ctx* ctx, double* b, int32_t p);
std::vector<double> residual_norms(adp_ctx* ctx, const adp_csr* a, const double* v, int64_t ld, int32_t e,
                                   const std::vector<double>& lam, double* av);

// host symmetric eigensolver for small matrices (Jacobi; host_eig.cpp): a is
// column-major p x p, overwritten; returns ascending eigenvalues, vectors in z.
std::vector<double> host_sym_eig(std::vector<double>& a, int p, std::vector<double>& z);

}  // namespace adp
