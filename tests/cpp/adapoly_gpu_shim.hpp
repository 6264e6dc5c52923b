// The reference-side binding of INTEGRATION.md, verbatim: what a maintainer adds to the reference
// (e.g. proj/src/cheb_filter_gpu.hpp) to route clenshaw_apply / maspmm to libadp_b200.so. It includes the
// REFERENCE's own headers (adapoly/...) and include/adp.h; tests/cpp/ref_shim_test.cpp compiles it against
// the reference tree and checks it bitwise against the reference's CPU functions.
#pragma once

#include <stdexcept>
#include <string>

#include "adapoly/cheb_filter.hpp"
#include "adapoly/types.hpp"
#include "adp.h"

namespace adapoly::gpu {

// adp_status -> the reference exception types (types.hpp:23-46)
inline void check(adp_status s) {
  if (s == ADP_OK) return;
  const std::string m = adp_last_error_message();
  switch (s) {
    case ADP_ERR_CONFIG: throw ConfigError(m);
    case ADP_ERR_DIMENSION: throw DimensionError(m);
    case ADP_ERR_NOT_PD: throw NotPositiveDefinite(m);
    case ADP_ERR_PARSE: throw ParseError(m, 0);
    default: throw std::runtime_error(m);
  }
}

struct Device {  // one per process/GPU
  adp_ctx* ctx = nullptr;
  explicit Device(int dev = 0) { check(adp_ctx_create(dev, &ctx)); }
  ~Device() { adp_ctx_destroy(ctx); }
};

struct DeviceMatrix {  // replaces TiledMatrixd; built once per solve (solver.cpp:153)
  adp_csr* h = nullptr;
  DeviceMatrix(Device& d, const CsrMatrixd& a) {
    check(adp_csr_create(d.ctx, a.n_rows, a.n_cols, a.row_ptr.data(), a.col_idx.data(), a.values.data(), ADP_F64, &h));
  }
  ~DeviceMatrix() { adp_csr_destroy(h); }
};

inline Matrixd clenshaw_apply(Device& d, const ChebFilter& f, const DeviceMatrix& a,
                              const Eigen::Ref<const Matrixd>& x, int degree, std::int64_t* spmv_count = nullptr) {
  Matrixd y(x.rows(), x.cols());
  check(adp_filter_apply(d.ctx, a.h, f.coeffs.data(), f.k_max, f.l1, f.l2, degree, x.data(), x.rows(),
                         x.outerStride(), x.cols(), ADP_COL_MAJOR, y.data(), y.rows(), spmv_count));
  return y;
}

// maspmm: C += A B on column-major Eigen matrices
inline void maspmm(Device& d, const DeviceMatrix& a, const Matrixd& b, Matrixd& c) {
  check(adp_spmm(d.ctx, a.h, b.data(), b.rows(), b.outerStride(), b.cols(), ADP_COL_MAJOR, c.data(), c.outerStride(),
                 /*accumulate=*/1));
}

}  // namespace adapoly::gpu
