// C-ABI implementation of the operator level: context, device CSR, the
// Clenshaw filter application and maspmm (include/adp.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <utility>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

int64_t block_ld(int64_t q, bool cplx) {
  static const int64_t align = [] {  // fp64 columns; 32 = one 256-byte panel
    const char* e = std::getenv("ADP_WS_ALIGN");
    const int64_t v = e ? std::atoll(e) : 32;
    return v >= 2 && v % 2 == 0 ? v : 32;
  }();
  const int64_t m = cplx ? std::max<int64_t>(align / 2, 1) : align;  // elements per alignment unit
  if (q > m) return (q + m - 1) / m * m;
  return cplx ? q : ((q + 1) / 2) * 2;
}

namespace {
thread_local std::string g_last_error;

template <class F>
adp_status guarded(F&& f) {
  try {
    f();
    return ADP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("host allocation failed: ") + e.what();
    return ADP_ERR_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ADP_ERR_RUNTIME;
  }
}

size_t elem_bytes(const adp_csr* a) { return a->dtype == ADP_C128 ? 16 : 8; }

// Row-major workspace leading dimension: even number of fp64 columns so every
// row starts 16-byte aligned; complex rows are already 16-byte elements.
// Blocks wider than one 256-byte panel round up to whole panels: every row (and every 32-column
// panel of it) then starts on a 256-byte boundary -- with p = 926 columns (7408-byte rows) the sweep
// kernel's TMA boxes straddle cache lines (ADP_WS_ALIGN=2 restores the minimal pitch for A/B timing).
int64_t ws_ld(const adp_csr* a, int64_t q) { return block_ld(q, a->dtype == ADP_C128); }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

void set_device(adp_ctx* ctx) { ADP_CUDA(cudaSetDevice(ctx->device)); }

// Degree after dropping exactly-zero trailing coefficients (cheb_filter.cpp:141-142).
int effective_degree(const double* coeffs, int degree) {
  int deg = degree;
  while (deg > 0 && coeffs[deg] == 0.0) --deg;
  return deg;
}

// The device core of clenshaw_apply (cheb_filter.cpp:146-178) on row-major
// blocks. Y: input (ld_y), out: result (ld_out), w_buf / v_buf: workspaces
// with leading dimension ld. Degree already reduced.
void clenshaw_device(adp_ctx* ctx, const adp_csr* a, const double* coeffs, double l1, double l2, int deg,
                     const void* y, int64_t ld_y, void* out, int64_t ld_out, void* w_buf, void* v_buf, int64_t ld,
                     int64_t q) {
  const int eb = static_cast<int>(elem_bytes(a));
  const int64_t n = a->n_rows;
  if (deg == 0) {  // f.coeffs[0] * x
    launch_scale_rows(ctx, y, ld_y, out, ld_out, n, q, coeffs[0], eb);
    return;
  }
  StepArgs s{};
  s.a = a;
  s.q = q;
  s.row_begin = 0;
  s.row_end = n;
  s.goff = 0;
  if (deg == 1) {  // c0 x + c1 (l1 A x + l2 x)
    s.gsrc = y;
    s.ld = ld_y;
    s.ld_y = ld_y;
    s.out = out;
    s.ld_out = ld_out;
    s.s0 = coeffs[0];
    s.s1 = coeffs[1];
    s.s2 = l1;
    s.s3 = l2;
    launch_step(ctx, StepMode::Deg1, s);
    return;
  }
  // w = c_d y ; v = 2 l1 A w + (2 l2 + c_{d-1}/c_d) w ; swap(v, w)
  s.gsrc = y;
  s.ld = ld_y;
  s.ld_y = ld_y;
  s.wout = w_buf;
  s.out = v_buf;
  s.ld_out = ld;
  s.s0 = 2.0 * l1;
  s.s1 = 2.0 * l2 + coeffs[deg - 1] / coeffs[deg];
  s.s2 = coeffs[deg];
  launch_step(ctx, StepMode::First, s);
  void* cur_w = v_buf;
  void* cur_v = w_buf;
  s.wout = nullptr;
  s.yin = y;
  s.ld = ld;
  s.ld_y = ld_y;
  // Steps j = deg-2 .. 1: v = ((2l1 A w + 2l2 w) - v) + c_j y ; swap. Step 0 (the
  // last): v = ((l1 A w + l2 w) - v) + c0 y, written straight to the output.
  auto scalars = [&](int j, double* t) {
    t[0] = j == 0 ? l1 : 2.0 * l1;
    t[1] = j == 0 ? l2 : 2.0 * l2;
    t[2] = coeffs[j];
  };
  int j = deg - 2;
  for (; j >= 0; --j) {
    s.gsrc = cur_w;
    s.vin = cur_v;
    s.out = j == 0 ? out : cur_v;
    s.ld_out = j == 0 ? ld_out : ld;
    double t[3];
    scalars(j, t);
    s.s0 = t[0];
    s.s1 = t[1];
    s.s2 = t[2];
    launch_step(ctx, StepMode::Step, s);
    std::swap(cur_w, cur_v);
  }
}

void check_filter_args(const adp_csr* a, const double* coeffs, int32_t k_max, int32_t degree, int64_t x_rows,
                       int64_t q) {
  if (!a) fail(ADP_ERR_RUNTIME, "clenshaw_apply: null matrix");
  if (degree < 0 || degree > k_max) fail(ADP_ERR_CONFIG, "clenshaw_apply: degree out of range");
  if (!coeffs) fail(ADP_ERR_CONFIG, "clenshaw_apply: null coefficient array");
  if (x_rows != a->n_cols) fail(ADP_ERR_DIMENSION, "clenshaw_apply: operand row count does not match A");
  if (a->n_rows != a->n_cols) fail(ADP_ERR_DIMENSION, "clenshaw_apply: operator must be square");
  if (q < 0) fail(ADP_ERR_DIMENSION, "clenshaw_apply: negative column count");
}

// host (layout, ld) -> device row-major (ldd), via staging for column-major.
void upload_block(adp_ctx* ctx, const void* host, int64_t n, int64_t q, int64_t ldh, adp_layout layout, void* dev,
                  int64_t ldd, void* staging, size_t eb) {
  if (n == 0 || q == 0) return;
  if (layout == ADP_ROW_MAJOR) {
    ADP_CUDA(cudaMemcpy2DAsync(dev, ldd * eb, host, ldh * eb, q * eb, n, cudaMemcpyHostToDevice, ctx->stream));
    return;
  }
  if (ldh == n)
    ADP_CUDA(cudaMemcpyAsync(staging, host, n * q * eb, cudaMemcpyHostToDevice, ctx->stream));
  else
    ADP_CUDA(cudaMemcpy2DAsync(staging, n * eb, host, ldh * eb, n * eb, q, cudaMemcpyHostToDevice, ctx->stream));
  launch_colmajor_to_rowmajor(ctx, staging, n, q, n, dev, ldd, static_cast<int>(eb));
}

void download_block(adp_ctx* ctx, const void* dev, int64_t ldd, int64_t n, int64_t q, void* host, int64_t ldh,
                    adp_layout layout, void* staging, size_t eb) {
  if (n == 0 || q == 0) return;
  if (layout == ADP_ROW_MAJOR) {
    ADP_CUDA(cudaMemcpy2DAsync(host, ldh * eb, dev, ldd * eb, q * eb, n, cudaMemcpyDeviceToHost, ctx->stream));
    return;
  }
  launch_rowmajor_to_colmajor(ctx, dev, n, q, ldd, staging, n, static_cast<int>(eb));
  if (ldh == n)
    ADP_CUDA(cudaMemcpyAsync(host, staging, n * q * eb, cudaMemcpyDeviceToHost, ctx->stream));
  else
    ADP_CUDA(cudaMemcpy2DAsync(host, ldh * eb, staging, n * eb, n * eb, q, cudaMemcpyDeviceToHost, ctx->stream));
}

// The host-API filter on a large block, pipelined over column chunks (columns are independent:
// every chunk's result is bitwise the whole call's): chunk k + 1's H2D copy and layout transpose
// run on a copy stream while chunk k filters on the context's stream, and chunk k's transpose back
// and D2H copy overlap chunk k + 1's filter. Device memory: 6 chunk blocks instead of 4 full blocks.
void filter_apply_pipelined(adp_ctx* ctx, const adp_csr* a, const double* coeffs, double l1, double l2, int deg,
                            const void* x, int64_t ldx, int64_t q, adp_layout layout, void* y, int64_t ldy,
                            size_t eb) {
  const int64_t n = a->n_rows;
  const int64_t cw = std::min<int64_t>(q, ((q + 3) / 4 + 63) / 64 * 64);  // ~4 chunks, whole 64-column panels
  const int64_t nchunks = (q + cw - 1) / cw;
  const int64_t ld = ws_ld(a, cw);
  const size_t blk = static_cast<size_t>(n) * ld * eb, stg = static_cast<size_t>(n) * cw * eb;
  char* yb[2] = {static_cast<char*>(ctx->ws[1].get(blk)), static_cast<char*>(ctx->ws[4].get(blk))};
  void* wbuf = ctx->ws[2].get(blk);
  void* vbuf = ctx->ws[3].get(blk);
  char* st_in[2];
  char* st_out[2];
  char* stage = static_cast<char*>(ctx->ws[0].get(4 * stg));
  for (int i = 0; i < 2; ++i) {
    st_in[i] = stage + i * stg;
    st_out[i] = stage + (2 + i) * stg;
  }
  if (!ctx->copy_stream) ADP_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  cudaStream_t cs = ctx->copy_stream, ms = ctx->stream;
  std::vector<cudaEvent_t> ev;
  auto event = [&]() {
    cudaEvent_t e;
    ADP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
    return e;
  };
  struct Guard {
    std::vector<cudaEvent_t>& ev;
    ~Guard() {
      for (auto e : ev) cudaEventDestroy(e);
    }
  } guard{ev};
  cudaEvent_t start = event();
  ADP_CUDA(cudaEventRecord(start, ms));  // the copy stream starts after the caller's prior work
  ADP_CUDA(cudaStreamWaitEvent(cs, start, 0));
  const char* xh = static_cast<const char*>(x);
  char* yh = static_cast<char*>(y);
  std::vector<cudaEvent_t> up(nchunks), comp(nchunks), ready(nchunks), down(nchunks);
  for (int64_t k = 0; k < nchunks; ++k) {
    up[k] = event();
    comp[k] = event();
    ready[k] = event();
    down[k] = event();
  }
  auto upload = [&](int64_t k) {  // host chunk k -> yb[k % 2] (copy stream)
    const int64_t c0 = k * cw, qc = std::min(cw, q - c0);
    if (k >= 2) ADP_CUDA(cudaStreamWaitEvent(cs, comp[k - 2], 0));  // yb[k % 2] free
    struct OnCopyStream {  // the layout kernels of the upload run on the copy stream
      adp_ctx* c;
      cudaStream_t saved;
      ~OnCopyStream() { c->stream = saved; }
    } on{ctx, ms};
    ctx->stream = cs;
    if (ld != qc) ADP_CUDA(cudaMemsetAsync(yb[k % 2], 0, blk, cs));
    if (layout == ADP_COL_MAJOR)
      upload_block(ctx, xh + c0 * ldx * eb, n, qc, ldx, layout, yb[k % 2], ld, st_in[k % 2], eb);
    else
      upload_block(ctx, xh + c0 * eb, n, qc, ldx, layout, yb[k % 2], ld, st_in[k % 2], eb);
    ADP_CUDA(cudaEventRecord(up[k], cs));
  };
  upload(0);
  for (int64_t k = 0; k < nchunks; ++k) {
    const int64_t c0 = k * cw, qc = std::min(cw, q - c0);
    if (k + 1 < nchunks) upload(k + 1);
    ADP_CUDA(cudaStreamWaitEvent(ms, up[k], 0));
    void* obuf = (deg % 2 == 0) ? wbuf : vbuf;
    clenshaw_device(ctx, a, coeffs, l1, l2, deg, yb[k % 2], ld, obuf, ld, wbuf, vbuf, ld, qc);
    ADP_CUDA(cudaEventRecord(comp[k], ms));
    // transpose out on the compute stream (before the next chunk reuses W / V), then D2H on the copy stream
    if (k >= 2) ADP_CUDA(cudaStreamWaitEvent(ms, down[k - 2], 0));  // st_out[k % 2] free
    char* host_k = layout == ADP_COL_MAJOR ? yh + c0 * ldy * eb : yh + c0 * eb;
    if (layout == ADP_COL_MAJOR) {
      launch_rowmajor_to_colmajor(ctx, obuf, n, qc, ld, st_out[k % 2], n, static_cast<int>(eb));
      ADP_CUDA(cudaEventRecord(ready[k], ms));
      ADP_CUDA(cudaStreamWaitEvent(cs, ready[k], 0));
      if (ldy == n)
        ADP_CUDA(cudaMemcpyAsync(host_k, st_out[k % 2], n * qc * eb, cudaMemcpyDeviceToHost, cs));
      else
        ADP_CUDA(cudaMemcpy2DAsync(host_k, ldy * eb, st_out[k % 2], n * eb, n * eb, qc, cudaMemcpyDeviceToHost, cs));
    } else {
      ADP_CUDA(cudaMemcpy2DAsync(st_out[k % 2], qc * eb, obuf, ld * eb, qc * eb, n, cudaMemcpyDeviceToDevice, ms));
      ADP_CUDA(cudaEventRecord(ready[k], ms));
      ADP_CUDA(cudaStreamWaitEvent(cs, ready[k], 0));
      ADP_CUDA(cudaMemcpy2DAsync(host_k, ldy * eb, st_out[k % 2], qc * eb, qc * eb, n, cudaMemcpyDeviceToHost, cs));
    }
    ADP_CUDA(cudaEventRecord(down[k], cs));
  }
  ADP_CUDA(cudaStreamSynchronize(cs));
  ADP_CUDA(cudaStreamSynchronize(ms));
}

}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }

}  // namespace adp

using namespace adp;

extern "C" {

int32_t adp_version(void) { return 1; }

const char* adp_last_error_message(void) { return adp::g_last_error.c_str(); }

adp_status adp_ctx_create(int32_t device, adp_ctx** out) {
  return guarded([&] {
    int count = 0;
    ADP_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) fail(ADP_ERR_CONFIG, "adp_ctx_create: no such device");
    auto* ctx = new adp_ctx;
    ctx->device = device;
    try {
      ADP_CUDA(cudaSetDevice(device));
      ADP_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
      ADP_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
    } catch (...) {
      delete ctx;
      throw;
    }
    ctx->stream = ctx->own_stream;
    const char* no_pdl = std::getenv("ADP_NO_PDL");
    ctx->pdl = !(no_pdl && no_pdl[0] == '1');
    const char* no_line = std::getenv("ADP_NO_LINE");
    ctx->auto_line = !(no_line && no_line[0] == '1');
    const char* no_cube = std::getenv("ADP_NO_CUBE");
    ctx->auto_cube = !(no_cube && no_cube[0] == '1');
    const char* no_sweep = std::getenv("ADP_NO_SWEEP");
    ctx->auto_sweep = !(no_sweep && no_sweep[0] == '1');
    const char* no_band = std::getenv("ADP_NO_BAND");
    ctx->auto_band = !(no_band && no_band[0] == '1');
    *out = ctx;
  });
}

void adp_release_dense_handles(adp_ctx* ctx);  // dense.cu (extern "C")

adp_status adp_ctx_destroy(adp_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    adp_release_dense_handles(ctx);
    for (auto& b : ctx->ws) b.release();
    if (ctx->halo_failed) cudaFree(ctx->halo_failed);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
  });
}

adp_status adp_ctx_set_stream(adp_ctx* ctx, void* stream) {
  return guarded([&] {
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

void* adp_ctx_own_stream(const adp_ctx* ctx) { return ctx ? static_cast<void*>(ctx->own_stream) : nullptr; }

adp_status adp_ctx_synchronize(adp_ctx* ctx) {
  return guarded([&] {
    set_device(ctx);
    ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int64_t adp_ctx_launch_count(const adp_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t adp_ctx_last_step_kernel(const adp_ctx* ctx) { return ctx ? ctx->last_kernel : 0; }

adp_status adp_csr_stencil(adp_csr* a, int32_t* kind, int64_t* dims) {
  return guarded([&] {
    if (!a || !kind || !dims) fail(ADP_ERR_CONFIG, "adp_csr_stencil: null argument");
    set_device(a->ctx);
    const adp::StencilPlan* p = a->dtype == ADP_F64 && a->nnz <= 27 * a->n_rows ? adp::get_stencil_plan(a) : nullptr;
    *kind = p && p->valid ? p->kind : 0;
    dims[0] = p && p->valid ? p->nx : 0;
    dims[1] = p && p->valid ? p->ny : 0;
    dims[2] = p && p->valid ? p->nz : 0;
  });
}

adp_status adp_ctx_set_panel(adp_ctx* ctx, int32_t panel_cols) {
  return guarded([&] {
    if (panel_cols < 0) fail(ADP_ERR_CONFIG, "adp_ctx_set_panel: negative panel width");
    ctx->panel_cols = panel_cols;
  });
}

adp_status adp_ctx_set_tuning(adp_ctx* ctx, int32_t variant) {
  return guarded([&] {
    // 0 automatic; 1-5 force one kernel family (adp.h)
    if (variant < 0 || variant > 11) fail(ADP_ERR_CONFIG, "adp_ctx_set_tuning: unknown variant");
    ctx->variant = variant;
  });
}

// csr upload; validation mirrors CsrMatrix::validate (csr_matrix.hpp:101-116).
adp_status adp_csr_create(adp_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                          const int64_t* col_idx, const void* values, adp_dtype dtype, adp_csr** out) {
  return guarded([&] {
    if (n_rows < 0 || n_cols < 0) fail(ADP_ERR_DIMENSION, "negative matrix size");
    if (n_cols > std::numeric_limits<int32_t>::max() || n_rows > std::numeric_limits<int32_t>::max())
      fail(ADP_ERR_DIMENSION, "adp_csr_create: dimension exceeds int32 column indexing");
    if (dtype != ADP_F64 && dtype != ADP_C128) fail(ADP_ERR_CONFIG, "adp_csr_create: unknown dtype");
    if (row_ptr[0] != 0) fail(ADP_ERR_DIMENSION, "row_ptr endpoints mismatch");
    const int64_t nnz = row_ptr[n_rows];
    std::vector<int32_t> col32(static_cast<size_t>(nnz));
    for (int64_t r = 0; r < n_rows; ++r) {
      if (row_ptr[r + 1] < row_ptr[r]) fail(ADP_ERR_DIMENSION, "row_ptr not non-decreasing");
      for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
        if (col_idx[k] < 0 || col_idx[k] >= n_cols) fail(ADP_ERR_DIMENSION, "column index out of range");
        if (k > row_ptr[r] && col_idx[k] <= col_idx[k - 1])
          fail(ADP_ERR_DIMENSION, "columns not strictly increasing within a row");
        col32[k] = static_cast<int32_t>(col_idx[k]);
      }
    }
    set_device(ctx);
    auto* a = new adp_csr;
    a->ctx = ctx;
    a->device = ctx->device;
    a->n_rows = n_rows;
    a->n_cols = n_cols;
    a->nnz = nnz;
    a->dtype = dtype;
    // int64 row offsets when nnz >= 2^31 (config 5); ADP_FORCE_RP64=1 selects them for any size so
    // the 64-bit path is testable on small operators (tests/test_gpu_parity.py).
    const char* force64 = std::getenv("ADP_FORCE_RP64");
    a->rp64 = nnz > std::numeric_limits<int32_t>::max() || (force64 && force64[0] == '1');
    const size_t eb = dtype == ADP_C128 ? 16 : 8;
    try {
      const size_t rp_bytes = (n_rows + 1) * (a->rp64 ? 8 : 4);
      ADP_CUDA(cudaMalloc(&a->row_ptr, rp_bytes));
      ADP_CUDA(cudaMalloc(reinterpret_cast<void**>(&a->col_idx), std::max<size_t>(nnz, 1) * 4));
      ADP_CUDA(cudaMalloc(&a->values, std::max<size_t>(nnz, 1) * eb));
      if (a->rp64) {
        ADP_CUDA(cudaMemcpy(a->row_ptr, row_ptr, rp_bytes, cudaMemcpyHostToDevice));
      } else {
        std::vector<int32_t> rp32(n_rows + 1);
        for (int64_t r = 0; r <= n_rows; ++r) rp32[r] = static_cast<int32_t>(row_ptr[r]);
        ADP_CUDA(cudaMemcpy(a->row_ptr, rp32.data(), rp_bytes, cudaMemcpyHostToDevice));
      }
      if (nnz) {
        ADP_CUDA(cudaMemcpy(a->col_idx, col32.data(), nnz * 4, cudaMemcpyHostToDevice));
        ADP_CUDA(cudaMemcpy(a->values, values, nnz * eb, cudaMemcpyHostToDevice));
      }
      adp::plan_uploads_done();  // pageable copies may return before their DMA lands (adp_internal.hpp)
      a->h_row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
      a->h_col = std::move(col32);
      a->h_values = std::malloc(std::max<size_t>(nnz, 1) * eb);
      if (!a->h_values) throw std::bad_alloc();
      if (nnz) std::memcpy(a->h_values, values, nnz * eb);
      a->host_ready = true;
    } catch (...) {
      std::free(a->h_values);
      cudaFree(a->row_ptr);
      cudaFree(a->col_idx);
      cudaFree(a->values);
      delete a;
      throw;
    }
    *out = a;
  });
}

adp_status adp_csr_create_device(adp_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* d_row_ptr,
                                 const int32_t* d_col_idx, const void* d_values, adp_dtype dtype, adp_csr** out) {
  return guarded([&] {
    if (n_rows < 0 || n_cols < 0 || nnz < 0) fail(ADP_ERR_DIMENSION, "negative matrix size");
    if (n_cols > std::numeric_limits<int32_t>::max() || n_rows > std::numeric_limits<int32_t>::max())
      fail(ADP_ERR_DIMENSION, "adp_csr_create_device: dimension exceeds int32 column indexing");
    if (dtype != ADP_F64 && dtype != ADP_C128) fail(ADP_ERR_CONFIG, "adp_csr_create_device: unknown dtype");
    set_device(ctx);
    const int bad = adp::validate_csr_device(ctx, d_row_ptr, d_col_idx, n_rows, n_cols, nnz);
    if (bad & 1) fail(ADP_ERR_DIMENSION, "row_ptr not non-decreasing from 0 to nnz");
    if (bad & 2) fail(ADP_ERR_DIMENSION, "column index out of range");
    if (bad & 4) fail(ADP_ERR_DIMENSION, "columns not strictly increasing within a row");
    auto* a = new adp_csr;
    a->ctx = ctx;
    a->device = ctx->device;
    a->n_rows = n_rows;
    a->n_cols = n_cols;
    a->nnz = nnz;
    a->dtype = dtype;
    const char* force64 = std::getenv("ADP_FORCE_RP64");
    a->rp64 = nnz > std::numeric_limits<int32_t>::max() || (force64 && force64[0] == '1');
    const size_t eb = dtype == ADP_C128 ? 16 : 8;
    try {
      const size_t rp_bytes = (n_rows + 1) * (a->rp64 ? 8 : 4);
      ADP_CUDA(cudaMalloc(&a->row_ptr, rp_bytes));
      ADP_CUDA(cudaMalloc(reinterpret_cast<void**>(&a->col_idx), std::max<size_t>(nnz, 1) * 4));
      ADP_CUDA(cudaMalloc(&a->values, std::max<size_t>(nnz, 1) * eb));
      if (a->rp64)
        ADP_CUDA(cudaMemcpyAsync(a->row_ptr, d_row_ptr, rp_bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      else
        adp::narrow_row_ptr_device(ctx, d_row_ptr, static_cast<int32_t*>(a->row_ptr), n_rows + 1);
      if (nnz) {
        ADP_CUDA(cudaMemcpyAsync(a->col_idx, d_col_idx, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
        ADP_CUDA(cudaMemcpyAsync(a->values, d_values, nnz * eb, cudaMemcpyDeviceToDevice, ctx->stream));
      }
      ADP_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      cudaFree(a->row_ptr);
      cudaFree(a->col_idx);
      cudaFree(a->values);
      delete a;
      throw;
    }
    *out = a;
  });
}


adp_status adp_csr_destroy(adp_csr* a) {
  return guarded([&] {
    if (!a) return;
    cudaSetDevice(a->device);  // cudaFree waits for work still using the buffers
    cudaFree(a->row_ptr);
    cudaFree(a->col_idx);
    cudaFree(a->values);
    std::free(a->h_values);
    delete a;
  });
}

adp_status adp_csr_info(const adp_csr* a, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, int32_t* dtype) {
  return guarded([&] {
    if (n_rows) *n_rows = a->n_rows;
    if (n_cols) *n_cols = a->n_cols;
    if (nnz) *nnz = a->nnz;
    if (dtype) *dtype = a->dtype;
  });
}

adp_status adp_filter_apply_device(adp_ctx* ctx, const adp_csr* a, const double* coeffs, int32_t k_max, double l1,
                                   double l2, int32_t degree, const void* dx, int64_t x_rows, int64_t ldx, int64_t q,
                                   void* dy, int64_t ldy, int64_t* spmv_count) {
  return guarded([&] {
    check_filter_args(a, coeffs, k_max, degree, x_rows, q);
    if (q == 0) return;
    if (ldx < q || ldy < q) fail(ADP_ERR_DIMENSION, "clenshaw_apply: leading dimension smaller than q");
    set_device(ctx);
    const int deg = effective_degree(coeffs, degree);
    if (spmv_count) *spmv_count += static_cast<int64_t>(deg) * q;
    const size_t eb = elem_bytes(a);
    const int64_t n = a->n_rows;
    const int64_t ld = ws_ld(a, q);
    // Operands that already satisfy the kernel contract are used in place:
    // 16-byte aligned rows and no padding column that the last vector would
    // touch (q even for fp64).
    const bool pad_free = a->dtype == ADP_C128 || q % 2 == 0;
    const bool x_ok = pad_free && aligned16(dx) && (a->dtype == ADP_C128 || ldx % 2 == 0);
    const bool y_ok = pad_free && aligned16(dy) && (a->dtype == ADP_C128 || ldy % 2 == 0);
    const size_t blk = static_cast<size_t>(n) * ld * eb;
    const void* yin = dx;
    int64_t ld_y = ldx;
    if (!x_ok) {
      void* ybuf = ctx->ws[1].get(blk);
      ADP_CUDA(cudaMemsetAsync(ybuf, 0, blk, ctx->stream));
      ADP_CUDA(cudaMemcpy2DAsync(ybuf, ld * eb, dx, ldx * eb, q * eb, n, cudaMemcpyDeviceToDevice, ctx->stream));
      yin = ybuf;
      ld_y = ld;
    }
    void* wbuf = ctx->ws[2].get(blk);
    void* vbuf = ctx->ws[3].get(blk);
    if (y_ok) {
      clenshaw_device(ctx, a, coeffs, l1, l2, deg, yin, ld_y, dy, ldy, wbuf, vbuf, ld, q);
    } else {
      void* obuf = ctx->ws[4].get(blk);
      clenshaw_device(ctx, a, coeffs, l1, l2, deg, yin, ld_y, obuf, ld, wbuf, vbuf, ld, q);
      ADP_CUDA(cudaMemcpy2DAsync(dy, ldy * eb, obuf, ld * eb, q * eb, n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
  });
}

adp_status adp_filter_apply(adp_ctx* ctx, const adp_csr* a, const double* coeffs, int32_t k_max, double l1,
                            double l2, int32_t degree, const void* x, int64_t x_rows, int64_t ldx, int64_t q,
                            adp_layout layout, void* y, int64_t ldy, int64_t* spmv_count) {
  return guarded([&] {
    check_filter_args(a, coeffs, k_max, degree, x_rows, q);
    if (q == 0) return;
    const int64_t n = a->n_rows;
    if (layout == ADP_COL_MAJOR ? (ldx < n || ldy < n) : (ldx < q || ldy < q))
      fail(ADP_ERR_DIMENSION, "clenshaw_apply: leading dimension too small");
    set_device(ctx);
    const int deg = effective_degree(coeffs, degree);
    if (spmv_count) *spmv_count += static_cast<int64_t>(deg) * q;
    const size_t eb = elem_bytes(a);
    if (deg >= 2 && q >= 256 && static_cast<size_t>(n) * q * eb >= (size_t{1} << 30)) {
      // large blocks: column chunks with their host copies overlapped with the previous chunk's filter
      filter_apply_pipelined(ctx, a, coeffs, l1, l2, deg, x, ldx, q, layout, y, ldy, eb);
      return;
    }
    const int64_t ld = ws_ld(a, q);
    const size_t blk = static_cast<size_t>(n) * ld * eb;
    void* staging = ctx->ws[0].get(static_cast<size_t>(n) * q * eb);
    void* ybuf = ctx->ws[1].get(blk);
    void* wbuf = ctx->ws[2].get(blk);
    void* vbuf = ctx->ws[3].get(blk);
    if (ld != q) ADP_CUDA(cudaMemsetAsync(ybuf, 0, blk, ctx->stream));
    upload_block(ctx, x, n, q, ldx, layout, ybuf, ld, staging, eb);
    // The result lands in the V workspace of the last step (in place), then
    // leaves through the staging buffer.
    void* obuf = deg >= 2 ? ((deg % 2 == 0) ? wbuf : vbuf) : vbuf;
    clenshaw_device(ctx, a, coeffs, l1, l2, deg, ybuf, ld, obuf, ld, wbuf, vbuf, ld, q);
    download_block(ctx, obuf, ld, n, q, y, ldy, layout, staging, eb);
    ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adp_status adp_step_device(adp_ctx* ctx, const adp_csr* a, int32_t mode, const void* g, int64_t ld,
                           const void* vin, const void* yin, int64_t ld_y, void* out, void* wout, int64_t ld_out,
                           int64_t q, int64_t row_begin, int64_t row_end, int64_t goff, double s0, double s1,
                           double s2, double s3) {
  return guarded([&] {
    if (mode < 0 || mode > 4) fail(ADP_ERR_CONFIG, "adp_step_device: unknown mode");
    if (row_begin < 0 || row_end > a->n_rows || row_begin > row_end)
      fail(ADP_ERR_DIMENSION, "adp_step_device: row range outside the operator");
    if (q < 0 || ld < q || ld_out < q || (mode == 1 && ld_y < q))
      fail(ADP_ERR_DIMENSION, "adp_step_device: leading dimension smaller than q");
    set_device(ctx);
    StepArgs s{};
    s.a = a;
    s.gsrc = g;
    s.vin = vin;
    s.yin = yin;
    s.out = out;
    s.wout = wout;
    s.ld = ld;
    s.ld_y = mode == 1 ? ld_y : ld;
    s.ld_out = ld_out;
    s.q = q;
    s.row_begin = row_begin;
    s.row_end = row_end;
    s.goff = goff;
    s.s0 = s0;
    s.s1 = s1;
    s.s2 = s2;
    s.s3 = s3;
    launch_step(ctx, static_cast<StepMode>(mode), s);
  });
}

namespace {
std::vector<adp::PushTarget> push_targets(int64_t eb, const adp_halo_target* t, int32_t n) {
  if (n < 0 || n > adp::kMaxPush) fail(ADP_ERR_CONFIG, "halo: at most 4 push targets");
  std::vector<adp::PushTarget> out(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    if (!t[i].dst || t[i].ld < 0 || t[i].row_lo < 0 || t[i].row_hi < t[i].row_lo)
      fail(ADP_ERR_DIMENSION, "halo: bad push target");
    if (t[i].ld * eb >= (int64_t{1} << 32)) fail(ADP_ERR_DIMENSION, "halo: target leading dimension too large");
    out[i] = adp::PushTarget{static_cast<char*>(t[i].dst), t[i].row_lo, t[i].row_hi, t[i].row_shift,
                             static_cast<uint32_t>(t[i].ld * eb)};
  }
  return out;
}
}  // namespace

adp_status adp_step_device_push(adp_ctx* ctx, const adp_csr* a, int32_t mode, const void* g, int64_t ld,
                                const void* vin, const void* yin, int64_t ld_y, void* out, void* wout, int64_t ld_out,
                                int64_t q, int64_t row_begin, int64_t row_end, int64_t goff, double s0, double s1,
                                double s2, double s3, const adp_halo_target* targets, int32_t n_targets) {
  return guarded([&] {
    if (mode != 0 && mode != 1) fail(ADP_ERR_CONFIG, "adp_step_device_push: First / Step modes only");
    if (row_begin < 0 || row_end > a->n_rows || row_begin > row_end)
      fail(ADP_ERR_DIMENSION, "adp_step_device_push: row range outside the operator");
    if (q < 0 || ld < q || ld_out < q || (mode == 1 && ld_y < q))
      fail(ADP_ERR_DIMENSION, "adp_step_device_push: leading dimension smaller than q");
    const std::vector<adp::PushTarget> pt = push_targets(a->dtype == ADP_C128 ? 16 : 8, targets, n_targets);
    set_device(ctx);
    StepArgs s{};
    s.a = a;
    s.gsrc = g;
    s.vin = vin;
    s.yin = yin;
    s.out = out;
    s.wout = wout;
    s.ld = ld;
    s.ld_y = mode == 1 ? ld_y : ld;
    s.ld_out = ld_out;
    s.q = q;
    s.row_begin = row_begin;
    s.row_end = row_end;
    s.goff = goff;
    s.s0 = s0;
    s.s1 = s1;
    s.s2 = s2;
    s.s3 = s3;
    s.push = pt.data();
    s.n_push = n_targets;
    launch_step(ctx, static_cast<StepMode>(mode), s);
  });
}

adp_status adp_halo_push_rows(adp_ctx* ctx, adp_dtype dtype, const void* src, int64_t ld, int64_t row_begin,
                              int64_t row_end, int64_t q, const adp_halo_target* targets, int32_t n_targets) {
  return guarded([&] {
    if (dtype != ADP_F64 && dtype != ADP_C128) fail(ADP_ERR_CONFIG, "adp_halo_push_rows: unknown dtype");
    const int64_t eb = dtype == ADP_C128 ? 16 : 8;
    const std::vector<adp::PushTarget> pt = push_targets(eb, targets, n_targets);
    set_device(ctx);
    adp::launch_push_rows(ctx, src, ld * eb, row_begin, row_end, q * eb, pt.data(), n_targets);
  });
}

adp_status adp_halo_signal(adp_ctx* ctx, uint64_t* const* remote_counters, int32_t n, uint64_t value) {
  return guarded([&] {
    set_device(ctx);
    adp::launch_halo_signal(ctx, remote_counters, n, value);
  });
}

adp_status adp_halo_wait(adp_ctx* ctx, const uint64_t* const* local_counters, int32_t n, uint64_t expected,
                         uint32_t timeout_ms) {
  return guarded([&] {
    set_device(ctx);
    adp::launch_halo_wait(ctx, local_counters, n, expected, timeout_ms);
  });
}

adp_status adp_halo_check(adp_ctx* ctx) {
  return guarded([&] {
    if (!ctx->halo_failed) return;
    set_device(ctx);
    int h = 0;
    ADP_CUDA(cudaMemcpyAsync(&h, ctx->halo_failed, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ADP_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h) {
      ADP_CUDA(cudaMemsetAsync(ctx->halo_failed, 0, sizeof(int), ctx->stream));
      fail(ADP_ERR_NCCL, "halo exchange: a neighbour did not signal within the timeout");
    }
  });
}

adp_status adp_ipc_handle(const void* dptr, void* handle_out) {
  return guarded([&] {
    cudaIpcMemHandle_t h;
    ADP_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
    std::memcpy(handle_out, &h, sizeof(h));
  });
}

adp_status adp_ipc_open(int32_t device, const void* handle, void** dptr_out) {
  return guarded([&] {
    ADP_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    ADP_CUDA(cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

adp_status adp_ipc_close(void* dptr) {
  return guarded([&] { ADP_CUDA(cudaIpcCloseMemHandle(dptr)); });
}

adp_status adp_spmm_device(adp_ctx* ctx, const adp_csr* a, const void* db, int64_t b_rows, int64_t ldb, int64_t k,
                           void* dc, int64_t ldc, int32_t accumulate) {
  return guarded([&] {
    if (b_rows != a->n_cols) fail(ADP_ERR_DIMENSION, "maspmm: shape mismatch");
    if (k == 0) return;
    if (ldb < k || ldc < k) fail(ADP_ERR_DIMENSION, "maspmm: leading dimension smaller than k");
    set_device(ctx);
    const size_t eb = elem_bytes(a);
    const bool pad_free = a->dtype == ADP_C128 || k % 2 == 0;
    const bool b_ok = pad_free && aligned16(db) && (a->dtype == ADP_C128 || ldb % 2 == 0);
    const bool c_ok = pad_free && aligned16(dc) && (a->dtype == ADP_C128 || ldc % 2 == 0);
    const int64_t ld = ws_ld(a, k);
    const void* bsrc = db;
    int64_t ld_b = ldb;
    if (!b_ok) {
      const size_t blk = static_cast<size_t>(a->n_cols) * ld * eb;
      void* bbuf = ctx->ws[1].get(blk);
      ADP_CUDA(cudaMemsetAsync(bbuf, 0, blk, ctx->stream));
      ADP_CUDA(cudaMemcpy2DAsync(bbuf, ld * eb, db, ldb * eb, k * eb, a->n_cols, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
      bsrc = bbuf;
      ld_b = ld;
    }
    void* cdst = dc;
    int64_t ld_c = ldc;
    const size_t cblk = static_cast<size_t>(a->n_rows) * ld * eb;
    if (!c_ok) {
      cdst = ctx->ws[4].get(cblk);
      ld_c = ld;
      if (accumulate) {
        ADP_CUDA(cudaMemsetAsync(cdst, 0, cblk, ctx->stream));
        ADP_CUDA(cudaMemcpy2DAsync(cdst, ld * eb, dc, ldc * eb, k * eb, a->n_rows, cudaMemcpyDeviceToDevice,
                                   ctx->stream));
      }
    }
    StepArgs s{};
    s.a = a;
    s.gsrc = bsrc;
    s.ld = ld_b;
    s.ld_y = ld_b;
    s.out = cdst;
    s.ld_out = ld_c;
    s.q = k;
    s.row_begin = 0;
    s.row_end = a->n_rows;
    launch_step(ctx, accumulate ? StepMode::SpmmAcc : StepMode::Spmm, s);
    if (!c_ok)
      ADP_CUDA(cudaMemcpy2DAsync(dc, ldc * eb, cdst, ld * eb, k * eb, a->n_rows, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
  });
}

adp_status adp_spmm(adp_ctx* ctx, const adp_csr* a, const void* b, int64_t b_rows, int64_t ldb, int64_t k,
                    adp_layout layout, void* c, int64_t ldc, int32_t accumulate) {
  return guarded([&] {
    if (b_rows != a->n_cols) fail(ADP_ERR_DIMENSION, "maspmm: shape mismatch");
    if (k == 0) return;
    set_device(ctx);
    const size_t eb = elem_bytes(a);
    const int64_t ld = ws_ld(a, k);
    const int64_t nb = a->n_cols, nc = a->n_rows;
    void* staging = ctx->ws[0].get(static_cast<size_t>(std::max(nb, nc)) * k * eb);
    void* bbuf = ctx->ws[1].get(static_cast<size_t>(nb) * ld * eb);
    void* cbuf = ctx->ws[4].get(static_cast<size_t>(nc) * ld * eb);
    if (ld != k) {
      ADP_CUDA(cudaMemsetAsync(bbuf, 0, static_cast<size_t>(nb) * ld * eb, ctx->stream));
      ADP_CUDA(cudaMemsetAsync(cbuf, 0, static_cast<size_t>(nc) * ld * eb, ctx->stream));
    }
    upload_block(ctx, b, nb, k, ldb, layout, bbuf, ld, staging, eb);
    if (accumulate) upload_block(ctx, c, nc, k, ldc, layout, cbuf, ld, staging, eb);
    StepArgs s{};
    s.a = a;
    s.gsrc = bbuf;
    s.ld = ld;
    s.ld_y = ld;
    s.out = cbuf;
    s.ld_out = ld;
    s.q = k;
    s.row_begin = 0;
    s.row_end = nc;
    launch_step(ctx, accumulate ? StepMode::SpmmAcc : StepMode::Spmm, s);
    download_block(ctx, cbuf, ld, nc, k, c, ldc, layout, staging, eb);
    ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adp_status adp_fill_gaussian_device(adp_ctx* ctx, double* d_out, int64_t n, int64_t q, int64_t ld, uint64_t seed,
                                    uint64_t stream) {
  return guarded([&] {
    set_device(ctx);
    launch_fill_philox(ctx, d_out, n, q, ld, seed, stream, 0);
  });
}

adp_status adp_fill_rademacher_device(adp_ctx* ctx, double* d_out, int64_t n, int64_t q, int64_t ld,
                                      uint64_t seed, uint64_t stream) {
  return guarded([&] {
    set_device(ctx);
    launch_fill_philox(ctx, d_out, n, q, ld, seed, stream, 1);
  });
}

}  // extern "C"
