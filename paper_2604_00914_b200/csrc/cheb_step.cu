// Fused Clenshaw-step CSR SpMM kernel for sm_100a (B200).
//
// One launch = one degree step of clenshaw_apply (reference:
// proj/src/cheb_filter.cpp:162-177), i.e. one maspmm (proj/include/adapoly/
// tiled_matrix.hpp:184-210) fused with the elementwise recurrence update and
// the coefficient accumulation that the reference runs as separate Eigen array
// passes (plus aw.set_zero()). Per step the kernel streams W (gathered through
// A's column indices; L2 absorbs the stencil reuse), V (read + write in place)
// and Y (read): 4 n x q blocks, the algorithmic minimum.
//
// Mapping: a "task" is (row r, column panel). A group of G threads (G = 32: one
// warp) owns the task; lane l holds CH 16-byte vectors of the panel (2 fp64
// columns or 1 complex128 column each), so every gathered W row panel is read
// as fully coalesced 16 B-per-lane loads. The group walks row r's nonzeros in
// CSR order (ascending column) -- the reference's per-element accumulation
// order -- broadcasting (col, val) with shuffles and keeping U rows of loads in
// flight. The epilogue operands V[r], Y[r] are prefetched into shared memory
// with cp.async (LDGSTS) at task start so their latency hides under the
// gathers without costing registers.
//
// Arithmetic uses __dmul_rn/__dadd_rn/__dsub_rn only (never FMA), in the exact
// expression order of the reference, so results are bit-identical to the CPU
// reference (x86-64 SSE2, no FMA) -- see tests/test_gpu_parity.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "adp_internal.hpp"

namespace adp {
namespace {

constexpr int kThreads = 256;

struct KArgs {
  const void* row_ptr;
  const int32_t* col;
  const void* val;
  const double2* g;    // gathered operand
  const double2* vin;
  const double2* yin;
  double2* out;
  double2* wout;
  int64_t ldv;      // leading dimension of g/vin in 16-byte vectors
  int64_t ldyv;     // leading dimension of yin in 16-byte vectors
  int64_t ldo;      // leading dimension of out/wout in 16-byte vectors
  int64_t qv;       // number of 16-byte vectors per row holding real data (ceil)
  int64_t row_begin;
  int64_t nrows;
  int64_t n_panels;
  int64_t goff;           // row r's own row in g is r + goff (halo-extended layouts)
  double s0, s1, s2, s3;
};

// ---- scalar fields --------------------------------------------------------------
struct RealF {
  using Val = double;
  static __device__ __forceinline__ Val load_val(const void* p, int64_t k) {
    return __ldg(static_cast<const double*>(p) + k);
  }
  static __device__ __forceinline__ Val shfl(unsigned mask, Val v, int src, int width) {
    return __shfl_sync(mask, v, src, width);
  }
  static __device__ __forceinline__ Val zero() { return 0.0; }
  // acc += v * w (reference: cseg[t] += v * bseg[t], tiled_matrix.hpp:205)
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};

struct CplxF {
  using Val = double2;
  static __device__ __forceinline__ Val load_val(const void* p, int64_t k) {
    return __ldg(static_cast<const double2*>(p) + k);
  }
  static __device__ __forceinline__ Val shfl(unsigned mask, Val v, int src, int width) {
    Val o;
    o.x = __shfl_sync(mask, v.x, src, width);
    o.y = __shfl_sync(mask, v.y, src, width);
    return o;
  }
  static __device__ __forceinline__ Val zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    // complex128 has no reference implementation: its accumulation is defined
    // as four fused multiply-adds per entry (oracle.cpp cplx mac, std::fma), half the FP64
    // instructions of mul + add -- config 5 is FP64-issue bound
    acc.x = __fma_rn(v.x, w.x, acc.x);
    acc.x = __fma_rn(-v.y, w.y, acc.x);
    acc.y = __fma_rn(v.x, w.y, acc.y);
    acc.y = __fma_rn(v.y, w.x, acc.y);
    return acc;
  }
};

__device__ __forceinline__ double2 scale2(double s, double2 a) {
  return make_double2(__dmul_rn(s, a.x), __dmul_rn(s, a.y));
}
__device__ __forceinline__ double2 add2(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 sub2(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// Streaming operands (V, Y, the output) are touched once per step: mark them
// evict-first in L2 so the 126 MB L2 is left to the gathered W rows, whose
// stencil reuse distance (one grid plane) is what the cache must cover.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <class RP>
__device__ __forceinline__ int64_t load_rp(const void* p, int64_t i) {
  return static_cast<int64_t>(__ldg(static_cast<const RP*>(p) + i));
}

// ---- the kernel -------------------------------------------------------------------
// G threads per task, CH 16-byte vectors per thread (panel = G*CH vectors), U
// gathered rows in flight per batch, MINB resident blocks per SM requested from
// ptxas, HINT = evict-first L2 policy on the streaming operands.
template <class F, int G, int CH, int U, int MODE, class RP, int MINB, bool HINT>
__global__ void __launch_bounds__(kThreads, MINB) cheb_step_kernel(const KArgs p) {
  static_assert(kThreads % G == 0 && U <= G && G % U == 0, "bad tiling");
  constexpr int kTasksPerBlock = kThreads / G;
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;

  __shared__ double2 stage[kStep ? 2 * CH * kThreads : 1];

  const int lane = threadIdx.x % G;
  const unsigned mask =
      G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (((threadIdx.x & 31) / G) * G));
  const int64_t task = static_cast<int64_t>(blockIdx.x) * kTasksPerBlock + threadIdx.x / G;
  if (task >= p.nrows * p.n_panels) return;  // uniform within the group
  const int64_t panel = task / p.nrows;
  const int64_t r = p.row_begin + (task - panel * p.nrows);
  const int64_t cv0 = panel * (G * CH) + lane;  // vector column of chunk 0
  const int64_t rown = r + p.goff;              // own row inside the gathered operand
  uint64_t pol = 0;
  if constexpr (HINT) pol = evict_first_policy();

  bool cv[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) cv[c] = cv0 + c * G < p.qv;

  // Prefetch the epilogue operands V[r], Y[r] into shared memory (no registers).
  if constexpr (kStep) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (cv[c]) {
        double2* sv = &stage[(2 * c) * kThreads + threadIdx.x];
        double2* sy = &stage[(2 * c + 1) * kThreads + threadIdx.x];
        if constexpr (HINT) {
          cp_async16_hint(sv, p.vin + r * p.ldv + cv0 + c * G, pol);
          cp_async16_hint(sy, p.yin + r * p.ldyv + cv0 + c * G, pol);
        } else {
          cp_async16(sv, p.vin + r * p.ldv + cv0 + c * G);
          cp_async16(sy, p.yin + r * p.ldyv + cv0 + c * G);
        }
      }
    }
  }

  double2 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if constexpr (kSpmmAcc)
      acc[c] = cv[c] ? p.out[r * p.ldo + cv0 + c * G] : make_double2(0.0, 0.0);
    else
      acc[c] = make_double2(0.0, 0.0);
  }
  double2 own[CH];
  bool have_own = false;
#pragma unroll
  for (int c = 0; c < CH; ++c) own[c] = make_double2(0.0, 0.0);

  const int64_t start = load_rp<RP>(p.row_ptr, r);
  const int64_t end = load_rp<RP>(p.row_ptr, r + 1);
  for (int64_t base = start; base < end; base += G) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(G), end - base));
    int my_col = 0;
    typename F::Val my_val = F::zero();
    if (lane < cnt) {
      my_col = __ldg(p.col + base + lane);
      my_val = F::load_val(p.val, base + lane);
    }
    for (int k0 = 0; k0 < cnt; k0 += U) {
      double2 w[U][CH];
      int cidx[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        cidx[u] = __shfl_sync(mask, my_col, k0 + u, G);
        if (k0 + u < cnt) {
          const double2* src = p.g + static_cast<int64_t>(cidx[u]) * p.ldv + cv0;
#pragma unroll
          for (int c = 0; c < CH; ++c)
            if (cv[c]) w[u][c] = __ldg(src + c * G);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const typename F::Val v = F::shfl(mask, my_val, k0 + u, G);
        if (k0 + u < cnt) {
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            if (!cv[c]) continue;
            double2 wv = w[u][c];
            if constexpr (kFirst) wv = scale2(p.s2, wv);  // W = c_d * Y, materialised on the fly
            acc[c] = F::mac(acc[c], v, wv);
            if constexpr (kNeedOwn) {
              if (cidx[u] == rown) own[c] = wv;
            }
          }
          if constexpr (kNeedOwn) have_own |= (cidx[u] == rown);
        }
      }
    }
  }

  if constexpr (kNeedOwn) {
    if (!have_own) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (cv[c]) {
          double2 wv = __ldg(p.g + rown * p.ldv + cv0 + c * G);
          if constexpr (kFirst) wv = scale2(p.s2, wv);
          own[c] = wv;
        }
      }
    }
  }
  if constexpr (kStep) cp_async_wait_all();

#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if (!cv[c]) continue;
    double2* dst = p.out + r * p.ldo + cv0 + c * G;
    double2 res;
    if constexpr (kStep) {
      // v = (((s0 * aw) + (s1 * w)) - v) + (s2 * y)   (cheb_filter.cpp:170-171, 176-177)
      const double2 vv = stage[(2 * c) * kThreads + threadIdx.x];
      const double2 yy = stage[(2 * c + 1) * kThreads + threadIdx.x];
      res = add2(sub2(add2(scale2(p.s0, acc[c]), scale2(p.s1, own[c])), vv), scale2(p.s2, yy));
    } else if constexpr (kFirst) {
      // w = c_d * y ; v = (2 l1) * aw + (2 l2 + c_{d-1}/c_d) * w   (cheb_filter.cpp:162-165)
      double2* wdst = p.wout + r * p.ldo + cv0 + c * G;
      if constexpr (HINT) st_hint(wdst, own[c], pol);
      else *wdst = own[c];
      res = add2(scale2(p.s0, acc[c]), scale2(p.s1, own[c]));
    } else if constexpr (kDeg1) {
      // c0 * x + c1 * (l1 * ax + l2 * x)   (cheb_filter.cpp:154)
      res = add2(scale2(p.s0, own[c]), scale2(p.s1, add2(scale2(p.s2, acc[c]), scale2(p.s3, own[c]))));
    } else {
      res = acc[c];
    }
    if constexpr (HINT) st_hint(dst, res, pol);
    else *dst = res;
  }
}

template <class F, int G, int CH, int U, class RP, int MINB, bool HINT>
void launch_mode(adp_ctx* ctx, StepMode mode, const KArgs& k, int64_t tasks) {
  constexpr int kTasksPerBlock = kThreads / G;
  const int64_t blocks = (tasks + kTasksPerBlock - 1) / kTasksPerBlock;
  if (blocks > 0x7fffffffLL) fail(ADP_ERR_DIMENSION, "cheb_step: grid too large");
  const dim3 grid(static_cast<unsigned>(blocks));
  switch (mode) {
    case StepMode::First:
      cheb_step_kernel<F, G, CH, U, 0, RP, MINB, HINT><<<grid, kThreads, 0, ctx->stream>>>(k);
      break;
    case StepMode::Step:
      cheb_step_kernel<F, G, CH, U, 1, RP, MINB, HINT><<<grid, kThreads, 0, ctx->stream>>>(k);
      break;
    case StepMode::Deg1:
      cheb_step_kernel<F, G, CH, U, 2, RP, MINB, HINT><<<grid, kThreads, 0, ctx->stream>>>(k);
      break;
    case StepMode::Spmm:
      cheb_step_kernel<F, G, CH, U, 3, RP, MINB, HINT><<<grid, kThreads, 0, ctx->stream>>>(k);
      break;
    case StepMode::SpmmAcc:
      cheb_step_kernel<F, G, CH, U, 4, RP, MINB, HINT><<<grid, kThreads, 0, ctx->stream>>>(k);
      break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

// Panel geometry for a full-warp group: n_panels panels of `ch` 32-vector chunks.
int64_t panels_for(int64_t qv, int64_t ch) { return (qv + 32 * ch - 1) / (32 * ch); }

template <class F, class RP>
void dispatch(adp_ctx* ctx, StepMode mode, KArgs k) {
  const int64_t qv = k.qv;
  if (qv <= 4) {
    k.n_panels = 1;
    launch_mode<F, 4, 1, 4, RP, 2, true>(ctx, mode, k, k.nrows);
    return;
  }
  if (qv <= 8) {
    k.n_panels = 1;
    launch_mode<F, 8, 1, 8, RP, 2, true>(ctx, mode, k, k.nrows);
    return;
  }
  if (qv <= 16) {
    k.n_panels = 1;
    launch_mode<F, 16, 1, 8, RP, 2, true>(ctx, mode, k, k.nrows);
    return;
  }
  auto go = [&](int64_t ch, auto launcher) {
    k.n_panels = panels_for(qv, ch);
    launcher(k.nrows * k.n_panels);
  };
  // <= 4 chunks per panel, balanced across panels
  const int64_t n_panels = (qv + 127) / 128;
  const int64_t ch = (((qv + n_panels - 1) / n_panels) + 31) / 32;
  switch (ch) {
    case 1: go(1, [&](int64_t t) { launch_mode<F, 32, 1, 8, RP, 3, true>(ctx, mode, k, t); }); break;
    case 2: go(2, [&](int64_t t) { launch_mode<F, 32, 2, 4, RP, 3, true>(ctx, mode, k, t); }); break;
    case 3: go(3, [&](int64_t t) { launch_mode<F, 32, 3, 4, RP, 2, true>(ctx, mode, k, t); }); break;
    default: go(4, [&](int64_t t) { launch_mode<F, 32, 4, 4, RP, 2, true>(ctx, mode, k, t); }); break;
  }
}

}  // namespace

namespace {
void launch_step_impl(adp_ctx* ctx, StepMode mode, const StepArgs& s);
}  // namespace

// Peer-memory halo push (multi-GPU row partition): the lean kernel stores the output rows a
// neighbour needs straight into its halo over NVLink from the epilogue that computed them.
// Other kernels (1-3 vectors, tuning variants) compute first and copy the rows out after.
void launch_step(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  // operand checks for every path (the halo-push fast path below included)
  const int epv = s.a->dtype == ADP_C128 ? 1 : 2;
  if (s.ld % epv || s.ld_out % epv || s.ld_y % epv)
    fail(ADP_ERR_DIMENSION, "cheb_step: leading dimension must be even for fp64");
  auto aligned = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; };
  if (!aligned(s.gsrc) || !aligned(s.out) || (s.vin && !aligned(s.vin)) || (s.yin && !aligned(s.yin)) ||
      (s.wout && !aligned(s.wout)))
    fail(ADP_ERR_DIMENSION, "cheb_step: operands must be 16-byte aligned");
  for (int t = 0; t < s.n_push; ++t)
    if ((reinterpret_cast<uintptr_t>(s.push[t].dst) & 15u) != 0 || s.push[t].ld_b % 16 != 0)
      fail(ADP_ERR_DIMENSION, "cheb_step: halo push targets must be 16-byte aligned");
  if (s.n_push == 0 || s.row_end <= s.row_begin || s.q == 0) return launch_step_impl(ctx, mode, s);
  if (mode != StepMode::First && mode != StepMode::Step) fail(ADP_ERR_CONFIG, "halo push: First / Step modes only");
  if (s.n_push > kMaxPush) fail(ADP_ERR_CONFIG, "halo push: too many targets");
  if ((ctx->variant == 0 || ctx->variant == 5) && launch_step_sweep(ctx, mode, s))
    return void(ctx->last_kernel = 5);
  if (ctx->variant == 0 && launch_step_lean(ctx, mode, s)) return void(ctx->last_kernel = 2);
  StepArgs t = s;
  t.push = nullptr;
  t.n_push = 0;
  launch_step_impl(ctx, mode, t);
  const int64_t eb = s.a->dtype == ADP_C128 ? 16 : 8;
  launch_push_rows(ctx, s.out, s.ld_out * eb, s.row_begin, s.row_end, s.q * eb, s.push, s.n_push);
}

namespace {
void launch_step_impl(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  const adp_csr* a = s.a;
  const bool cplx = a->dtype == ADP_C128;
  const int epv = cplx ? 1 : 2;
  if (s.row_end <= s.row_begin || s.q == 0) return;
  // Dispatch (variant 0 = automatic; adp_ctx_set_tuning forces one family):
  // the plane-sweep stencil kernel (cheb_sweep.cu) for Step launches on operators that are
  // a constant-coefficient 3-D stencil plus a diagonal; the band-block kernel (cheb_band.cu) for
  // banded operators with sparse off-band entries (config 5); the cube / line kernels for other
  // long-row stencils (cheb_cube.cu, cheb_line.cu); the lean kernel (cheb_lean.cu) for
  // >= 4 vectors; this file's narrow-group row kernel for 1-3 vectors and variant 1.
  const int v = ctx->variant;
  if ((v == 0 || v == 5) && launch_step_sweep(ctx, mode, s)) return void(ctx->last_kernel = 5);
  if ((v == 0 || (v >= 6 && v <= 11)) && launch_step_band(ctx, mode, s)) return void(ctx->last_kernel = 6);
  if (v == 4 && launch_step_cube(ctx, mode, s)) return void(ctx->last_kernel = 4);
  if ((v == 0 || v == 3) && launch_step_line(ctx, mode, s)) return void(ctx->last_kernel = 3);
  if (v != 1 && launch_step_lean(ctx, mode, s)) return void(ctx->last_kernel = 2);
  ctx->last_kernel = 1;
  KArgs k{};
  k.row_ptr = a->row_ptr;
  k.col = a->col_idx;
  k.val = a->values;
  k.g = static_cast<const double2*>(s.gsrc);
  k.vin = static_cast<const double2*>(s.vin);
  k.yin = static_cast<const double2*>(s.yin);
  k.out = static_cast<double2*>(s.out);
  k.wout = static_cast<double2*>(s.wout);
  k.ldv = s.ld / epv;
  k.ldo = s.ld_out / epv;
  k.ldyv = s.ld_y / epv;
  k.qv = (s.q + epv - 1) / epv;
  k.row_begin = s.row_begin;
  k.nrows = s.row_end - s.row_begin;
  k.goff = s.goff;
  k.s0 = s.s0;
  k.s1 = s.s1;
  k.s2 = s.s2;
  k.s3 = s.s3;
  if (cplx) {
    if (a->rp64) dispatch<CplxF, int64_t>(ctx, mode, k);
    else dispatch<CplxF, int32_t>(ctx, mode, k);
  } else {
    if (a->rp64) dispatch<RealF, int64_t>(ctx, mode, k);
    else dispatch<RealF, int32_t>(ctx, mode, k);
  }
}
}  // namespace

}  // namespace adp
