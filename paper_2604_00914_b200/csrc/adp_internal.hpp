// Internal definitions shared by the libadp_b200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "adp.h"

namespace adp {

using index_t = std::int64_t;

// Exceptions inside the library; the C-ABI converts them to adp_status.
struct Error : std::runtime_error {
  adp_status code;
  Error(adp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(adp_status c, const std::string& m) { throw Error(c, m); }

void set_last_error(const std::string& m);

#define ADP_CUDA(call)                                                                               \
  do {                                                                                               \
    cudaError_t err__ = (call);                                                                      \
    if (err__ != cudaSuccess)                                                                        \
      ::adp::fail(err__ == cudaErrorMemoryAllocation ? ADP_ERR_OOM : ADP_ERR_CUDA,                   \
                  std::string(#call) + ": " + cudaGetErrorString(err__));                            \
  } while (0)

#define ADP_LAUNCH_CHECK() ADP_CUDA(cudaGetLastError())

// Grow-only device scratch buffer.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      if (ptr) cudaFree(ptr);
      ptr = nullptr;
      bytes = 0;
      if (need) ADP_CUDA(cudaMalloc(&ptr, need));
      bytes = need;
    }
    return ptr;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

}  // namespace adp

struct adp_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // where work is queued (own or borrowed)
  cudaStream_t copy_stream = nullptr;  // host-API pipelining: chunk copies beside the filter (lazy)
  int sm_count = 148;
  int64_t launches = 0;
  int panel_cols = 0;  // 0 = automatic
  int variant = 0;     // kernel family (adp_ctx_set_tuning): 0 automatic, 1 row, 2 lean, 3 line, 4 cube, 5 sweep, 6 band
  bool pdl = true;        // programmatic dependent launch between degree steps (ADP_NO_PDL=1: off)
  bool auto_line = true;  // automatic line-kernel choice (ADP_NO_LINE=1: off, for A/B timing)
  bool auto_cube = true;  // automatic cube-kernel choice for its full panels (ADP_NO_CUBE=1: off)
  bool auto_sweep = true; // automatic plane-sweep stencil kernel (ADP_NO_SWEEP=1: off)
  bool auto_band = true;  // automatic band-block kernel (ADP_NO_BAND=1: off)
  int last_kernel = 0;    // family of the last step launch (adp_ctx_last_step_kernel)
  adp::DevBuf ws[6];   // scratch: staging, Y, W, V, misc
  void* cublas = nullptr;
  void* cusolver = nullptr;
  int* halo_failed = nullptr;  // set by the halo wait kernel on timeout (adp_halo_check)
};

namespace adp {
// Leading dimension (elements) of a row-major device block of q columns: 16-byte aligned rows, and
// whole 256-byte panels once the block is wider than one (ADP_WS_ALIGN overrides the fp64 column multiple).
int64_t block_ld(int64_t q, bool cplx);
// Shifted-pattern row blocks of an operator for the line kernel (cheb_line.cu).
struct LinePlan {
  int R = 0, mm = 0;
  bool band = false;          // band blocks allowed (register line kernel only)
  int64_t n_blocks = 0, n_regular = 0, n_patterns = 0, n_runs = 0, n_band = 0;
  double regular_frac = 0.0;
  void* d_blk_pat = nullptr;  // int32[n_blocks]: pattern id, -1 = row by row
  void* d_pat_ptr = nullptr;  // int32[n_patterns+1]: runs of each pattern
  void* d_runs = nullptr;     // int4[n_runs]: {first column - r0, entry index in the core, length, 0}
  // Band blocks: only a core of consecutive columns is shared (shifted by one per row); each row's
  // entries before it (prefix) and after it (suffix) run row by row. nullptr when no band block exists.
  void* d_prefix = nullptr;   // int32[n_rows]: entries before the core (0 outside band blocks)
  void* d_pat_len = nullptr;  // int32[n_patterns]: entries of each pattern's core
  ~LinePlan();
};
// Blocks of L = ly * lz lines of R consecutive rows (line l at r0 + off[l]) for the
// cube kernel (cheb_cube.cu): the union of the lines' column runs per shifted pattern.
constexpr int64_t kCubeValueSlot = 2048;  // bytes of shared memory per warp for a block's fp64 values (x2 complex)
struct CubePlan {
  int R = 0, ly = 0, lz = 0, mm = 0;
  int64_t row_begin = 0, row_end = 0;  // the rows the blocks cover (a launch's row range)
  bool valid = false;         // strides found and blocks built
  int64_t sy = 0, sz = 0;     // line strides derived from the dominant pattern
  int32_t off[8] = {};
  int64_t n_blocks = 0, n_regular = 0, n_rem = 0, n_patterns = 0, n_items = 0;
  double regular_rows_frac = 0.0;
  void* d_blk = nullptr;      // int4[n_blocks]: {r0, pattern, value offset lo, hi} (pattern -1: row by row, -2: r0 indexes the remainder list)
  void* d_pat_ptr = nullptr;  // int32[n_patterns+1]: items of each pattern
  void* d_pat_nv = nullptr;   // int32[n_patterns]: values per block of each pattern
  void* d_items = nullptr;    // int4[n_items]: {start - r0, length, line mask, 0}
  void* d_rem = nullptr;      // int32[n_rem]: rows outside every full block
  void* d_vals = nullptr;     // the regular blocks' values in kernel consumption order (item, line, row, position)
  ~CubePlan();
};
}  // namespace adp

namespace adp {
// A constant-coefficient stencil on a structured grid (cheb_sweep.cu): row r is grid point
// (x, y, z) = (r % nx, (r / nx) % ny, r / (nx ny)); its columns are the in-grid points of a fixed
// radius-1 offset set (the 27-point box or the 7-point star) in ascending order, and every row holds
// the same value at each offset except the centre (the diagonal: a potential), which is per row.
// Detected and verified entry by entry against the CSR once per operator; a lossless re-encoding.
struct StencilPlan {
  bool valid = false;
  int kind = 0;               // 27 (box) or 7 (star)
  int64_t nx = 0, ny = 0, nz = 0;  // nz: planes of the operator's rows
  int64_t nzw = 0;            // planes of the grid its columns index (> nz for a rank's halo-extended rows)
  int64_t goff = 0;           // row r is point r + goff of that grid
  int64_t nxp = 0;            // x pitch of the diagonal array (even: 16-byte rows for TMA)
  double w[27] = {};          // value at offset (dx, dy, dz): index (dz+1)*9 + (dy+1)*3 + (dx+1); centre unused
  bool classes = false;       // 27: weights depend only on m = |dx|+|dy|+|dz| (cls[m]); 7: all neighbours -1
  double cls[4] = {};
  double* d_diag = nullptr;   // [nz][ny][nxp] centre values
  std::string why;            // why the operator is not such a stencil (diagnostics)
  ~StencilPlan();
};
// A banded operator with sparse off-band entries (cheb_band.cu): every row r holds all columns
// max(0, r - h) .. min(n - 1, r + h), preceded by nlow[r] and followed by the rest of its entries.
struct BandPlan {
  bool valid = false;
  int64_t h = 0;
  int32_t* d_nlow = nullptr;  // [n] entries before the band
  ~BandPlan();
};
}  // namespace adp

struct adp_csr {
  adp_ctx* ctx = nullptr;     // creating context (must outlive every call that uses this operator)
  int device = 0;             // destroy needs only this: the operator may outlive its context
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  adp_dtype dtype = ADP_F64;
  bool rp64 = false;          // int64 row offsets (nnz >= 2^31)
  void* row_ptr = nullptr;    // int32[n_rows+1] or int64[n_rows+1]
  int32_t* col_idx = nullptr; // int32[nnz]
  void* values = nullptr;     // double[nnz] or double2[nnz]
  // host copies for the tiling preprocessing
  std::vector<int64_t> h_row_ptr;
  std::vector<int32_t> h_col;
  void* h_values = nullptr;  // malloc'd copy of the values
  bool host_ready = false;   // h_* filled (eagerly by adp_csr_create, lazily for device-created operators)
  std::vector<std::unique_ptr<adp::LinePlan>> line_plans;
  std::vector<std::unique_ptr<adp::CubePlan>> cube_plans;
  std::unique_ptr<adp::StencilPlan> stencil;  // built on first use (cheb_sweep.cu)
  std::unique_ptr<adp::BandPlan> band;        // built on first use (cheb_band.cu)
};

namespace adp {

// Launch with programmatic stream serialization (PDL) when the context allows
// it: the kernel must execute griddepcontrol.wait before reading anything the
// previous kernel on the stream writes.
template <class Kern, class... Args>
void launch_pdl(adp_ctx* ctx, Kern kern, dim3 grid, dim3 block, size_t smem, const Args&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ADP_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

// ---- kernels (cheb_step.cu) ---------------------------------------------------
enum class StepMode : int { First = 0, Step = 1, Deg1 = 2, Spmm = 3, SpmmAcc = 4 };

// One launch of the fused Clenshaw step: out = epilogue(A * G, own rows).
// A neighbour's rows of a halo-extended buffer, mapped into this process (CUDA IPC over
// NVLink): output row r in [lo, hi) is also stored at dst + (r + shift) * ld_b.
constexpr int kMaxPush = 4;
struct PushTarget {
  char* dst;
  int64_t lo, hi, shift;
  uint32_t ld_b;
};

struct StepArgs {
  const adp_csr* a;
  const void* gsrc;  // gathered operand (W for Step, Y for First, X for Deg1, B for Spmm)
  const void* vin;   // Step: V (previous), read
  const void* yin;   // Step: Y
  void* out;         // Step/Deg1/Spmm: output rows; First: V
  void* wout;        // First: W = c_d * Y
  int64_t ld;        // leading dimension (elements of the scalar type) of gsrc/vin
  int64_t ld_y;      // leading dimension of yin
  int64_t ld_out;    // leading dimension of out/wout
  int64_t q;         // columns
  int64_t row_begin, row_end;
  int64_t goff;      // own row of out-row r inside gsrc is r + goff (0 unless halo-extended)
  double s0, s1, s2, s3;
  const PushTarget* push = nullptr;  // First / Step: peer halo targets of the output rows (lean kernel)
  int32_t n_push = 0;
};
void launch_step(adp_ctx* ctx, StepMode mode, const StepArgs& args);
// Halo exchange over peer memory (layout.cu): copy rows [row_begin, row_end) of src that fall in a
// target's range to the target (then a system fence); signal: after every prior kernel on the stream,
// store `value` (release, system scope) to each remote counter; wait: spin (acquire, system scope)
// until every local counter >= expected (fails after ~timeout_ms rather than hanging the GPU).
void launch_push_rows(adp_ctx* ctx, const void* src, int64_t ld_b, int64_t row_begin, int64_t row_end,
                      int64_t row_bytes, const PushTarget* targets, int32_t n);
void launch_halo_signal(adp_ctx* ctx, uint64_t* const* counters, int32_t n, uint64_t value);
void launch_halo_wait(adp_ctx* ctx, const uint64_t* const* counters, int32_t n, uint64_t expected,
                      uint32_t timeout_ms);

// Layout kernels (layout.cu). Elements are 8 B (f64) or 16 B (c128).
void launch_colmajor_to_rowmajor(adp_ctx* ctx, const void* src, int64_t n, int64_t q, int64_t lds, void* dst,
                                 int64_t ldd, int elem_bytes);
void launch_rowmajor_to_colmajor(adp_ctx* ctx, const void* src, int64_t n, int64_t q, int64_t lds, void* dst,
                                 int64_t ldd, int elem_bytes);
void launch_scale_rows(adp_ctx* ctx, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t n, int64_t q,
                       double s, int elem_bytes);
void launch_fill_philox(adp_ctx* ctx, double* dst, int64_t n, int64_t q, int64_t ld, uint64_t seed,
                        uint64_t stream, int kind);

// The default lean kernel (cheb_lean.cu) for >= 4 vectors per row.
bool launch_step_lean(adp_ctx* ctx, StepMode mode, const StepArgs& args);

// The line kernel (cheb_line.cu): register reuse of gathered rows across
// blocks of rows with shifted column patterns. Returns false if not applicable.
bool launch_step_line(adp_ctx* ctx, StepMode mode, const StepArgs& args);
const LinePlan* get_line_plan(adp_csr* a, int rows_per_block, int max_run, bool band = false);
// The cube kernel (cheb_cube.cu): reuse across 2-D/3-D row blocks (tuning variants 111-118).
bool launch_step_cube(adp_ctx* ctx, StepMode mode, const StepArgs& args);
bool launch_cube_auto(adp_ctx* ctx, StepMode mode, const StepArgs& args, int64_t vectors);
const CubePlan* get_cube_plan(adp_csr* a, int rows_per_line, int ly, int lz, int max_run, int64_t row_begin,
                              int64_t row_end);
// The plane-sweep stencil kernel (cheb_sweep.cu): Step launches on constant-coefficient 3-D stencil
// operators (StencilPlan). Returns false if not applicable.
bool launch_step_sweep(adp_ctx* ctx, StepMode mode, const StepArgs& args);
const StencilPlan* get_stencil_plan(adp_csr* a, int64_t goff = 0);
// The band-block kernel (cheb_band.cu): Step launches on banded operators (config 5).
bool launch_step_band(adp_ctx* ctx, StepMode mode, const StepArgs& args);
const BandPlan* get_band_plan(adp_csr* a);
// Host copies of a device-created operator's arrays, downloaded on first use by the
// host-side preprocessing (line plans, tilings, segments, the dense fallback).
void ensure_host_copy(adp_csr* a);
// A host-built plan's arrays have been copied with cudaMemcpy from pageable memory, which may return
// before the DMA lands; kernels on the context's non-blocking stream are not ordered after it, so
// every plan builder waits for its uploads (on the legacy stream that carried them) before use.
inline void plan_uploads_done() { ADP_CUDA(cudaStreamSynchronize(cudaStreamLegacy)); }
// Device-side CSR validation (CsrMatrix::validate, csr_matrix.hpp:101-116): returns 0 if
// row_ptr is non-decreasing from 0 to nnz and every row's columns are strictly increasing in [0, n_cols).
int validate_csr_device(adp_ctx* ctx, const int64_t* row_ptr, const int32_t* col, int64_t n_rows, int64_t n_cols,
                        int64_t nnz);
void narrow_row_ptr_device(adp_ctx* ctx, const int64_t* src, int32_t* dst, int64_t count);

// Host filter helpers (filter_host.cpp).
std::vector<double> step_coeffs(double alpha, double beta, int k);
std::vector<double> lanczos_damping(int k, double m);
std::vector<double> jackson_damping(int k);
double map_clamped(const adp_filter_info& f, double x, bool* clamped);

}  // namespace adp
