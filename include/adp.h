/*
 * adp.h -- C-ABI drop-in boundary of the B200-native AdaPolySI Chebyshev-filter
 * hot path (libadp_b200.so).
 *
 * The reference (arxiv 2604.00914, /root/reference/proj) has no FFI layer: its
 * boundary is a set of C++ functions taking Eigen types. Each entry point below
 * replaces one of them; the comment names the reference declaration (file:line
 * relative to /root/reference/proj). Conventions:
 *   - plain pointers and sizes only, no C++ or torch types, no exceptions;
 *   - every call returns adp_status; the reference exception type maps 1:1 onto
 *     ADP_ERR_CONFIG / ADP_ERR_DIMENSION / ADP_ERR_NOT_PD / ADP_ERR_PARSE
 *     (include/adapoly/types.hpp:23-46); CUDA / NCCL / allocation failures get
 *     their own codes; adp_last_error_message() returns the message of the
 *     calling thread's last failure;
 *   - host dense operands default to column-major (Eigen's default storage,
 *     include/adapoly/types.hpp:13-20); device operands are row-major n x q with
 *     a leading dimension (the B200 kernel layout);
 *   - complex128 operands are interleaved (re, im) pairs (std::complex<double>);
 *   - calls are ordered on the context's stream and synchronise before returning
 *     host data. One host thread per context.
 */
#ifndef ADP_H_
#define ADP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ADP_OK = 0,
  ADP_ERR_CONFIG = 1,    /* adapoly::ConfigError        (types.hpp:40-42)   */
  ADP_ERR_DIMENSION = 2, /* adapoly::DimensionError     (types.hpp:36-38)   */
  ADP_ERR_NOT_PD = 3,    /* adapoly::NotPositiveDefinite (types.hpp:44-46)  */
  ADP_ERR_PARSE = 4,     /* adapoly::ParseError         (types.hpp:23-34)   */
  ADP_ERR_RUNTIME = 5,   /* std::runtime_error / std::invalid_argument      */
  ADP_ERR_CUDA = 6,      /* CUDA runtime / cuBLAS / cuSOLVER failure        */
  ADP_ERR_OOM = 7,       /* device allocation failed                        */
  ADP_ERR_NCCL = 8       /* collective failure (multi-GPU row partition)    */
} adp_status;

typedef enum { ADP_F64 = 0, ADP_C128 = 1 } adp_dtype;
typedef enum { ADP_COL_MAJOR = 0, ADP_ROW_MAJOR = 1 } adp_layout;
typedef enum { ADP_DAMP_LANCZOS = 0, ADP_DAMP_JACKSON = 1 } adp_damping;

typedef struct adp_ctx adp_ctx; /* device, stream, library handles, workspace */
typedef struct adp_csr adp_csr; /* device-resident CSR operator               */

/* ChebFilter minus its coefficient array (include/adapoly/cheb_filter.hpp:41-66). */
typedef struct {
  double interval_a, interval_b;
  double alpha, beta;
  int32_t k_max;
  double m;
  double l1, l2;
  double lambda_min, lambda_max;
  int32_t active_degree;
} adp_filter_info;

/* ---------------------------------------------------------------- context -- */
int32_t adp_version(void);
const char* adp_last_error_message(void);
adp_status adp_ctx_create(int32_t device, adp_ctx** out);
adp_status adp_ctx_destroy(adp_ctx* ctx);
/* Run all subsequent work of ctx on an existing cudaStream_t (e.g. torch's current
 * stream); NULL is the legacy default stream, as in any CUDA launch. */
adp_status adp_ctx_set_stream(adp_ctx* ctx, void* cuda_stream);
/* The non-blocking stream the context created for itself (its initial stream). */
void* adp_ctx_own_stream(const adp_ctx* ctx);
adp_status adp_ctx_synchronize(adp_ctx* ctx);
/* Number of kernels this library has launched on ctx (instrumentation for bench.py). */
int64_t adp_ctx_launch_count(const adp_ctx* ctx);
/* Kernel family of the last fused-step launch on ctx (1 row, 2 lean, 3 line, 4 cube,
 * 5 plane sweep, 6 band; 0 none yet) -- instrumentation for tests and bench.py. */
int32_t adp_ctx_last_step_kernel(const adp_ctx* ctx);
/* Kernel tuning knobs (0 = automatic): columns per warp task (panel width). */
adp_status adp_ctx_set_panel(adp_ctx* ctx, int32_t panel_cols);
/* Kernel family of the fused step kernel (0 = automatic). Every
 * family computes bit-identical results; they differ only in how the gathered
 * rows travel: 1 narrow-group row kernel, 2 lean kernel (one row per warp task),
 * 3 line kernel (register reuse across shifted-pattern row blocks), 4 cube kernel
 * (runs shared by 2-D/3-D blocks of grid lines), 5 plane-sweep stencil kernel
 * (constant-coefficient 3-D stencils: halo tiles of W streamed plane by plane
 * through shared memory), 6 band-block kernel (banded operators with sparse
 * off-band entries: W row panels shared by 8 consecutive rows, off-band rows
 * gathered through a cp.async ring), 7-11 the same with other block geometries
 * (4 / 6 / 8 rows, ring depths 2-4; measurement alternatives). A family that
 * does not apply to an operator falls back to the next one. Other values fail
 * with ADP_ERR_CONFIG. */
adp_status adp_ctx_set_tuning(adp_ctx* ctx, int32_t variant);

/* -------------------------------------------------------------- operator -- */
/* Upload a CSR matrix (CsrMatrix, include/adapoly/csr_matrix.hpp:22-117: int64
 * row_ptr / col_idx, columns strictly increasing within a row). Replaces
 * csr_to_tiled (include/adapoly/tiled_matrix.hpp:58-94): the device keeps CSR
 * with int32 column indices and int32 (nnz < 2^31) or int64 row offsets. Host
 * arrays are copied; the caller keeps ownership. values: double[nnz] or
 * interleaved complex128[nnz]. Columns must be sorted ascending per row: the
 * kernel accumulates in CSR order, which is the reference's ascending-column
 * order (tiled_matrix.hpp:78-81,200). */
adp_status adp_csr_create(adp_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                          const int64_t* col_idx, const void* values, adp_dtype dtype, adp_csr** out);
/* As adp_csr_create, from arrays already in device memory of ctx's device (a GPU-side
 * generator or loader: config 5's 2.16 G-nonzero operator never exists on the host).
 * d_row_ptr: int64[n_rows+1], d_col_idx: int32[nnz], d_values: double[nnz] or complex128[nnz].
 * Validated on the device like CsrMatrix::validate (csr_matrix.hpp:101-116): row_ptr
 * non-decreasing from 0 to nnz, columns strictly increasing within a row and in range.
 * The arrays are copied (the caller keeps and may free them after the call returns). */
adp_status adp_csr_create_device(adp_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* d_row_ptr,
                                 const int32_t* d_col_idx, const void* d_values, adp_dtype dtype, adp_csr** out);
adp_status adp_csr_destroy(adp_csr* a);
adp_status adp_csr_info(const adp_csr* a, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, int32_t* dtype);
/* Whether the operator is a constant-coefficient radius-1 stencil on a structured grid
 * (the plane-sweep kernel's precondition, verified entry by entry on first use):
 * kind = 27 (box) or 7 (star) with dims = {nx, ny, nz}, else kind = 0. */
adp_status adp_csr_stencil(adp_csr* a, int32_t* kind, int64_t* dims);

/* clenshaw_apply (include/adapoly/cheb_filter.hpp:84-86, src/cheb_filter.cpp:129-179):
 * Y = rho(l(A)) X with host X / Y. coeffs = ChebFilter::coeffs (k_max+1 doubles),
 * l1 / l2 = ChebFilter::l1 / l2. Same semantics as the reference: degree in
 * [0, k_max] else ADP_ERR_CONFIG; n_cols(A) != rows(X) -> ADP_ERR_DIMENSION;
 * trailing zero coefficients reduce the degree; degrees 0 / 1 use the direct
 * formulas; *spmv_count (if non-null) is incremented by effective_degree * q.
 * Bitwise identical to the reference's arithmetic (no FMA contraction). */
adp_status adp_filter_apply(adp_ctx* ctx, const adp_csr* a, const double* coeffs, int32_t k_max, double l1,
                            double l2, int32_t degree, const void* x, int64_t x_rows, int64_t ldx, int64_t q,
                            adp_layout layout, void* y, int64_t ldy, int64_t* spmv_count);
/* Same on device-resident row-major operands (x: n x q with leading dimension
 * ldx, y: n x q with ldy; y may alias nothing in x). Stream-ordered, no sync. */
adp_status adp_filter_apply_device(adp_ctx* ctx, const adp_csr* a, const double* coeffs, int32_t k_max, double l1,
                                   double l2, int32_t degree, const void* dx, int64_t x_rows, int64_t ldx, int64_t q,
                                   void* dy, int64_t ldy, int64_t* spmv_count);

/* One fused Clenshaw degree step on device row-major blocks, for drivers that
 * interleave steps with halo exchanges (multi-GPU row partition). mode:
 *   0 FIRST  w = s2*g[r] -> wout, out = s0*(A*(s2*g)) + s1*w     (cheb_filter.cpp:162-165)
 *   1 STEP   out = ((s0*(A*g) + s1*g[r]) - vin) + s2*yin          (cheb_filter.cpp:170-171,176-177)
 *   2 DEG1   out = s0*g[r] + s1*(s2*(A*g) + s3*g[r])              (cheb_filter.cpp:154)
 *   3 SPMM   out = A*g ;  4 SPMM_ACC out += A*g                   (tiled_matrix.hpp:184-210)
 * Rows [row_begin, row_end) of A; output row r lives at out + r*ld_out; the own
 * row of the gathered operand g is row r + goff (halo-extended layouts); all
 * column indices of A index rows of g. Stream-ordered, no synchronisation. */
adp_status adp_step_device(adp_ctx* ctx, const adp_csr* a, int32_t mode, const void* g, int64_t ld,
                           const void* vin, const void* yin, int64_t ld_y, void* out, void* wout, int64_t ld_out,
                           int64_t q, int64_t row_begin, int64_t row_end, int64_t goff, double s0, double s1,
                           double s2, double s3);

/* ------------------------------------------------ peer-memory halo exchange -- */
/* Multi-GPU row partition (the reference is single-process).
 * One process per GPU; each rank's halo-extended blocks are mapped into its neighbours
 * (CUDA IPC over NVLink). adp_step_device_push is adp_step_device (First / Step modes)
 * whose kernel ALSO stores every output row r in [row_lo, row_hi) to
 * dst + (r + row_shift) * ld (ld in scalar elements of the target rows): the rows a
 * neighbour needs land in its halo from the epilogue that computed them, with no
 * separate collective. adp_halo_signal then publishes (release, system scope) a step
 * count to each neighbour's counter after all prior work on the stream; adp_halo_wait
 * queues a wait (acquire, system scope) until every local counter >= expected -- the
 * next step's halo has landed -- failing (adp_halo_check -> ADP_ERR_NCCL) instead of
 * hanging after timeout_ms. adp_halo_push_rows copies rows already computed (the
 * filter's input block, narrow widths). adp_ipc_* wrap cudaIpc{Get,Open,Close}MemHandle
 * (64-byte handles). */
typedef struct {
  void* dst;
  int64_t row_lo, row_hi; /* rows of the local output block to push */
  int64_t row_shift;      /* local row r lands at target row r + row_shift */
  int64_t ld;             /* leading dimension of the target rows (scalar elements) */
} adp_halo_target;
adp_status adp_step_device_push(adp_ctx* ctx, const adp_csr* a, int32_t mode, const void* g, int64_t ld,
                                const void* vin, const void* yin, int64_t ld_y, void* out, void* wout, int64_t ld_out,
                                int64_t q, int64_t row_begin, int64_t row_end, int64_t goff, double s0, double s1,
                                double s2, double s3, const adp_halo_target* targets, int32_t n_targets);
adp_status adp_halo_push_rows(adp_ctx* ctx, adp_dtype dtype, const void* src, int64_t ld, int64_t row_begin,
                              int64_t row_end, int64_t q, const adp_halo_target* targets, int32_t n_targets);
adp_status adp_halo_signal(adp_ctx* ctx, uint64_t* const* remote_counters, int32_t n, uint64_t value);
adp_status adp_halo_wait(adp_ctx* ctx, const uint64_t* const* local_counters, int32_t n, uint64_t expected,
                         uint32_t timeout_ms);
adp_status adp_halo_check(adp_ctx* ctx);
adp_status adp_ipc_handle(const void* dptr, void* handle_out);
adp_status adp_ipc_open(int32_t device, const void* handle, void** dptr_out);
adp_status adp_ipc_close(void* dptr);

/* maspmm (include/adapoly/tiled_matrix.hpp:184-186): C += A B (accumulate != 0)
 * or C = A B (accumulate == 0; the reference's set_zero() + maspmm). Host
 * operands in the given layout; k = columns of B. */
adp_status adp_spmm(adp_ctx* ctx, const adp_csr* a, const void* b, int64_t b_rows, int64_t ldb, int64_t k,
                    adp_layout layout, void* c, int64_t ldc, int32_t accumulate);
adp_status adp_spmm_device(adp_ctx* ctx, const adp_csr* a, const void* db, int64_t b_rows, int64_t ldb, int64_t k,
                           void* dc, int64_t ldc, int32_t accumulate);

/* ---------------------------------------------- filter construction (host) -- */
/* chebyshev_step_coeffs (src/cheb_filter.cpp:21-37); out: k+1 doubles. */
adp_status adp_step_coeffs(double alpha, double beta, int32_t k, double* out);
/* lanczos_damping (src/cheb_filter.cpp:39-49) / jackson_damping (:51-61). */
adp_status adp_lanczos_damping(int32_t k, double m, double* out);
adp_status adp_jackson_damping(int32_t k, double* out);
/* build_filter (src/cheb_filter.cpp:63-94); coeffs: k+1 doubles. */
adp_status adp_build_filter(double a, double b, double lambda_min, double lambda_max, int32_t k, double m,
                            adp_damping damping, adp_filter_info* info, double* coeffs);
/* eval_filter_scalar (src/cheb_filter.cpp:96-127); *clamped (nullable) += clamp count. */
adp_status adp_eval_filter(const adp_filter_info* f, const double* coeffs, const double* x, int64_t n,
                           int32_t degree, double* out, int64_t* clamped);
/* initial_degree (src/cheb_filter.cpp:181-187). */
adp_status adp_initial_degree(double alpha, double beta, double c, int32_t* out);
/* adaptive_degree (src/cheb_filter.cpp:189-219). */
adp_status adp_adaptive_degree(const adp_filter_info* f, const double* coeffs, const double* ritz, int64_t p,
                               int64_t e_i, double tau_a, int32_t* out);

/* ------------------------------------------------------- filter bounds -- */
/* Truncation-error diagnostics of the damped step filter
 * (include/adapoly/filter_bounds.hpp:8-30, src/filter_bounds.cpp): J(theta),
 * the damping constant C_m (m > 0, else ADP_ERR_CONFIG), the pointwise
 * undamped (k >= 1) and damped (1 <= k_i <= k, m >= 0) bounds on |g - g_k|,
 * and the projector bound ||P - P_i||_2 from the eigenvalue angles
 * (non-empty, 1 <= k_i <= k_max). */
adp_status adp_j_theta(double theta, double alpha, double beta, double* out);
adp_status adp_c_m_constant(double m, double* out);
adp_status adp_undamped_bound(double theta, int32_t k, double alpha, double beta, double* out);
adp_status adp_damped_bound(double theta, int32_t k_i, int32_t k, double m, double alpha, double beta, double* out);
adp_status adp_projector_bound(const adp_filter_info* f, const double* thetas, int64_t count, int32_t k_i,
                               double* out);

/* ------------------------------------------------------------- seeded RNG -- */
/* fill_gaussian / fill_rademacher (include/adapoly/philox.hpp:92-109) into a
 * host column-major n x q buffer: Philox4x32-10, draw index c*n + r. */
adp_status adp_fill_gaussian(double* out, int64_t n, int64_t q, uint64_t seed, uint64_t stream);
adp_status adp_fill_rademacher(double* out, int64_t n, int64_t q, uint64_t seed, uint64_t stream);
/* Philox4x32-10 primitives (philox.hpp:25-72): gaussian / uniform draws
 * first..first+count-1 of (seed, stream), and one raw 4-word block. */
adp_status adp_philox_gaussian(uint64_t seed, uint64_t stream, uint64_t first, int64_t count, double* out);
adp_status adp_philox_uniform(uint64_t seed, uint64_t stream, uint64_t first, int64_t count, double* out);
adp_status adp_philox_block(uint64_t seed, uint64_t stream, uint64_t counter, uint32_t* out);
/* The same draws generated on the device into a row-major n x q block (ld). */
adp_status adp_fill_gaussian_device(adp_ctx* ctx, double* d_out, int64_t n, int64_t q, int64_t ld, uint64_t seed,
                                    uint64_t stream);
adp_status adp_fill_rademacher_device(adp_ctx* ctx, double* d_out, int64_t n, int64_t q, int64_t ld,
                                      uint64_t seed, uint64_t stream);

/* ------------------------------------------------- device solver subsystems -- */
/* csr_spmv (include/adapoly/csr_matrix.hpp:122-134): y = A x for real A, one row per thread,
 * products accumulated sequentially in CSR order (the Lanczos SpMV); device x, y. */
adp_status adp_spmv_device(adp_ctx* ctx, const adp_csr* a, const double* d_x, double* d_y);
/* estimate_spectrum_bounds (include/adapoly/lanczos.hpp:24-26, src/lanczos.cpp:81-111):
 * 40-step Lanczos with full reorthogonalisation on the device. */
adp_status adp_lanczos_bounds(adp_ctx* ctx, const adp_csr* a, int32_t steps, uint64_t seed, double* lambda_min,
                              double* lambda_max, int64_t* spmv_count);
/* estimate_eigcount (include/adapoly/solver.hpp:102-103, src/solver.cpp:108-117). */
adp_status adp_estimate_eigcount(adp_ctx* ctx, const adp_csr* a, const double* coeffs, int32_t k_max, double l1,
                                 double l2, int64_t probes, uint64_t seed, double* out, int64_t* spmv_count);
/* cholesky_qr (include/adapoly/dense_kernels.hpp:22, src/dense_kernels.cpp:53-92) in place on a
 * device row-major n x p block; *kept = orthonormal columns (dependent ones dropped, compacted). */
adp_status adp_cholesky_qr_device(adp_ctx* ctx, double* x, int64_t n, int64_t p, int64_t ld, int64_t* kept);
/* rayleigh_ritz (include/adapoly/dense_kernels.hpp:31, src/dense_kernels.cpp:94-101): theta
 * (host, ascending, qc doubles), V = Q U written to v_out (device row-major, ldv). */
adp_status adp_rayleigh_ritz_device(adp_ctx* ctx, const adp_csr* a, const double* q, int64_t ld, int64_t qc,
                                    double* theta, double* v_out, int64_t ldv);
/* compute_residuals (include/adapoly/solver.hpp:96-98, src/solver.cpp:94-106): norms (host). */
adp_status adp_residual_norms_device(adp_ctx* ctx, const adp_csr* a, const double* v, int64_t ld, int64_t e,
                                     const double* lambda, double* norms);
/* spurious_threshold (include/adapoly/solver.hpp:92, src/solver.cpp:81-92). */
adp_status adp_spurious_threshold(const double* ritz, int64_t n, double a, double b, double* out);

/* ------------------------------------------------------------------ solve -- */
/* SolverConfig (include/adapoly/solver.hpp:14-32); p_override <= 0 means "none".
 * tile_ti / tile_tk have no meaning on the device and are omitted. */
typedef struct {
  double interval_a, interval_b;
  double tau_c, tau_a, m, c, k_multiplier, mu;
  int64_t max_iter, lanczos_steps, trace_probes;
  uint64_t rng_seed;
  int64_t p_override;
  int32_t spurious_detection, collect_diagnostics;
} adp_solver_config;

/* IterationRecord (include/adapoly/solver.hpp:49-59). */
typedef struct {
  int64_t iteration;
  int32_t degree;
  int64_t active_width, e_in_interval, n_locked_total;
  double max_residual;
  int64_t spmv_filter, spmv_residual;
  double orth_error;
} adp_iteration_record;

/* StageTimings (include/adapoly/solver.hpp:61-68), seconds. */
typedef struct {
  double setup, filter, orth, rayleigh_ritz, residuals, other;
} adp_stage_timings;

/* SolveResult scalars (include/adapoly/solver.hpp:70-85). */
typedef struct {
  int64_t n, n_eigs, iterations, spmv_total, subspace_dim, n_history;
  int32_t converged, dense_fallback;
  double avg_degree, max_residual, e_estimate, lambda_min, lambda_max;
  adp_stage_timings timings;
} adp_solve_summary;

typedef struct adp_solve_result adp_solve_result;

void adp_solver_config_default(adp_solver_config* cfg);
/* solve (include/adapoly/solver.hpp:106, src/solver.cpp:119-360) on a real symmetric operator. */
adp_status adp_solve(adp_ctx* ctx, const adp_csr* a, const adp_solver_config* cfg, adp_solve_result** out);
adp_status adp_solve_summary_get(const adp_solve_result* r, adp_solve_summary* s);
/* eigenvalues ascending (n_eigs doubles); eigenvectors column-major n x n_eigs with ldv (either may be NULL). */
adp_status adp_solve_eigenpairs(const adp_solve_result* r, double* values, double* vectors, int64_t ldv);
/* n_history records and degrees (either may be NULL). */
adp_status adp_solve_history(const adp_solve_result* r, adp_iteration_record* records, int32_t* degree_history);
adp_status adp_solve_result_destroy(adp_solve_result* r);

#ifdef __cplusplus
}
#endif
#endif /* ADP_H_ */
