// The default fused Clenshaw-step kernel ("lean"), sm_100a.
//
// One degree step of clenshaw_apply (proj/src/cheb_filter.cpp:162-177: maspmm
// fused with the recurrence update and the coefficient accumulation), or a
// plain maspmm (tiled_matrix.hpp:184-210) in the Spmm modes.
//
// Mapping: a task = (row, column panel). A group of G lanes (G = 32: one warp;
// 16 / 8 / 4 for thin blocks) owns a task; lane l holds CH 16-byte vectors of
// the panel (2 fp64 columns or 1 complex128 column each), so each gathered W
// row panel is CH coalesced G*16-byte loads. Panels are always FULL (the
// dispatcher splits ragged widths into full-panel launches on column-offset
// pointers), so there are no per-vector predicates; index math is 32-bit with
// one IMAD.WIDE per gathered row.
//
// Memory: the epilogue operands V[r] and Y[r] arrive by TMA bulk copies
// (cp.async.bulk -> SASS UBLKCP, issued by the group's lane 0, L2 evict-first
// policy) into the group's shared-memory slot and complete on its mbarrier;
// results are stored with the same policy, leaving L2 to the gathered W rows
// whose stencil reuse it must cover. One gathered row in flight per group and
// many resident warps (64 registers, 4 blocks x 8 warps per SM for G = 32)
// measured fastest (profiles/r01_kernel_evolution.md).
//
// Arithmetic: __dmul_rn / __dadd_rn / __dsub_rn only, per row in CSR
// (ascending-column) order, in the reference's expression order: bitwise equal
// to the reference (x86-64 SSE2, no FMA).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <type_traits>

#include "adp_internal.hpp"

namespace adp {
namespace {

constexpr int kThreads = 256;

struct LArgs {
  const void* row_ptr;
  const int32_t* col;
  const void* val;
  const char* g;  // gathered operand (bytes)
  const char* vin;
  const char* yin;
  char* out;
  char* wout;
  uint32_t ldg_b, ldy_b, ldo_b;  // leading dimensions in bytes
  int64_t row_begin, nrows, n_panels, goff;
  int64_t g_rows;  // rows of the gathered operand (the operator's column count)
  int32_t valid;   // masked launches: vectors of the (single) panel that exist
  double s0, s1, s2, s3;
  // Peer-memory halo push (multi-GPU row partition, First / Step modes): output rows
  // r in [lo, hi) are also stored to dst + (r + shift) * ld_b, a neighbour's halo rows
  // of the same buffer mapped over NVLink (CUDA IPC), by the thread that computed them.
  PushTarget push[kMaxPush];
  int32_t n_push;
};

struct RealL {
  using Val = double;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double*>(p) + k); }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};
struct CplxL {
  using Val = double2;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double2*>(p) + k); }
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
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ uint64_t policy_evict_first(float frac) {
  uint64_t pol;  // runtime fraction operand: keeps ptxas from folding the policy
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, %1;\n" : "=l"(pol) : "f"(frac));
  return pol;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_hint(void* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
template <class RP>
__device__ __forceinline__ int64_t ld_rp(const void* p, int64_t i) {
  return static_cast<int64_t>(__ldg(static_cast<const RP*>(p) + i));
}
// Programmatic dependent launch: consecutive degree steps are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so this grid's CTAs can be
// resident while the previous step drains; nothing the previous step writes is
// read before griddepcontrol.wait (a no-op for ordinary launches). The next
// step may start launching as soon as every CTA of this one got here.
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

template <class F, int G, int CH, int U, int MODE, class RP, int MINB, bool MASK = false>
__global__ void __launch_bounds__(kThreads, MINB) cheb_lean_kernel(const LArgs p) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  constexpr int kGroups = kThreads / G;
  constexpr uint32_t kPB = G * CH * 16u;  // bytes of one row panel
  using Val = typename F::Val;
  extern __shared__ __align__(16) uint8_t smem[];  // [kGroups mbarriers][kGroups][V, Y] panels

  const int grp = threadIdx.x / G, lane = threadIdx.x % G;
  const int32_t nrows = static_cast<int32_t>(p.nrows);
  const int32_t task = static_cast<int32_t>(blockIdx.x) * kGroups + grp;
  if (task >= nrows * static_cast<int32_t>(p.n_panels)) return;  // group-uniform
  const int32_t panel = task / nrows;
  const int64_t r = p.row_begin + (task - panel * nrows);
  const uint32_t poff = static_cast<uint32_t>(panel) * kPB;
  const uint32_t voff = poff + lane * 16u;
  const uint64_t pol = policy_evict_first(1.0f);

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + grp;
  double2* my = reinterpret_cast<double2*>(smem + ((kGroups * 8 + 15) / 16) * 16) + grp * (2 * G * CH);
  const RP start = static_cast<RP>(ld_rp<RP>(p.row_ptr, r));  // the operator is constant: before the wait
  const RP end = static_cast<RP>(ld_rp<RP>(p.row_ptr, r + 1));
  pdl_wait_and_release();
  // masked launches (ragged widths): one panel whose vectors >= p.valid do not exist
  bool ok[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) ok[c] = !MASK || c * G + lane < p.valid;
  const uint32_t cpb = MASK ? static_cast<uint32_t>(p.valid) * 16u : kPB;  // bytes of the panel that exist
  if constexpr (kStep) {
    if (lane == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_arrive_expect_tx(bar, 2 * cpb);
      bulk_g2s_hint(my, p.vin + static_cast<uint64_t>(r) * p.ldg_b + poff, cpb, bar, pol);
      bulk_g2s_hint(my + G * CH, p.yin + static_cast<uint64_t>(r) * p.ldy_b + poff, cpb, bar, pol);
    }
  }
  char* ob = p.out + static_cast<uint64_t>(r) * p.ldo_b + voff;
  const char* gb = p.g + voff;

  double2 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if constexpr (kSpmmAcc)
      acc[c] = ok[c] ? *reinterpret_cast<const double2*>(ob + G * 16 * c) : make_double2(0.0, 0.0);
    else
      acc[c] = make_double2(0.0, 0.0);
  }
  for (RP e = start; e < end; e += U) {
    int cidx[U];
    Val v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (e + u < end) {
        cidx[u] = __ldg(p.col + e + u);
        v[u] = F::load(p.val, static_cast<int64_t>(e) + u);
      }
    }
    double2 w[U][CH];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (e + u < end) {
        const double2* src =
            reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cidx[u])) * p.ldg_b);
#pragma unroll
        for (int c = 0; c < CH; ++c) w[u][c] = ok[c] ? __ldg(src + G * c) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (e + u < end) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          double2 wv = w[u][c];
          if constexpr (kFirst) wv = scale2(p.s2, wv);  // W = c_d * Y, materialised on the fly
          acc[c] = F::mac(acc[c], v[u], wv);
        }
      }
    }
  }
  if constexpr (kStep) {
    __syncwarp();
    mbar_wait(bar, 0);
  }
  // own row of the gathered operand: an L1 hit (it was just gathered as the diagonal)
  const double2* own_src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(r + p.goff) * p.ldg_b);
  char* wb = kFirst ? p.wout + static_cast<uint64_t>(r) * p.ldo_b + voff : nullptr;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if (!ok[c]) continue;
    double2 own = make_double2(0.0, 0.0);
    if constexpr (kNeedOwn) own = __ldg(own_src + G * c);
    double2 res;
    if constexpr (kStep) {
      // v = (((s0 * aw) + (s1 * w)) - v) + (s2 * y)   (cheb_filter.cpp:170-171, 176-177)
      const double2 vv = my[c * G + lane];
      const double2 yy = my[G * CH + c * G + lane];
      res = add2(sub2(add2(scale2(p.s0, acc[c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
    } else if constexpr (kFirst) {
      // w = c_d * y ; v = (2 l1) * aw + (2 l2 + c_{d-1}/c_d) * w   (cheb_filter.cpp:162-165)
      const double2 wn = scale2(p.s2, own);
      st_hint(wb + G * 16 * c, wn, pol);
      res = add2(scale2(p.s0, acc[c]), scale2(p.s1, wn));
    } else if constexpr (kDeg1) {
      // c0 * x + c1 * (l1 * ax + l2 * x)   (cheb_filter.cpp:154)
      res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[c]), scale2(p.s3, own))));
    } else {
      res = acc[c];
    }
    st_hint(ob + G * 16 * c, res, pol);
    acc[c] = res;  // kept for the halo push below
  }
  if constexpr (kStep || kFirst) {
    // peer-memory halo: rows a neighbour needs also go straight into its block (one uniform
    // branch per row when not partitioned); then a system fence -- the peer's signal kernel
    // follows this grid in stream order, so the remote stores are performed before it runs
    if (p.n_push) {
      for (int t = 0; t < p.n_push; ++t) {
        if (r >= p.push[t].lo && r < p.push[t].hi) {
          char* dst = p.push[t].dst + static_cast<uint64_t>(r + p.push[t].shift) * p.push[t].ld_b + voff;
#pragma unroll
          for (int c = 0; c < CH; ++c)
            if (ok[c]) *reinterpret_cast<double2*>(dst + G * 16 * c) = acc[c];
        }
      }
      __threadfence_system();
    }
  }
}

template <class F, int G, int CH, int U, class RP, int MINB, bool MASK = false>
void launch_lean(adp_ctx* ctx, StepMode mode, LArgs k, int64_t qv) {
  constexpr int kGroups = kThreads / G;
  k.n_panels = MASK ? 1 : qv / (G * CH);
  k.valid = static_cast<int32_t>(qv);
  const int64_t total = k.nrows * k.n_panels;
  if (total >= (int64_t{1} << 31)) fail(ADP_ERR_DIMENSION, "cheb_lean: too many tasks");
  const int grid = static_cast<int>((total + kGroups - 1) / kGroups);
  const size_t smem = mode == StepMode::Step
                          ? static_cast<size_t>((kGroups * 8 + 15) / 16) * 16 + static_cast<size_t>(kGroups) * 2 * G * CH * 16
                          : 16;
  auto run = [&](auto kern) {
    if (smem > 48 * 1024)
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    launch_pdl(ctx, kern, dim3(grid), dim3(kThreads), smem, k);
  };
  switch (mode) {
    case StepMode::First: run(cheb_lean_kernel<F, G, CH, U, 0, RP, MINB, MASK>); break;
    case StepMode::Step: run(cheb_lean_kernel<F, G, CH, U, 1, RP, MINB, MASK>); break;
    case StepMode::Deg1: run(cheb_lean_kernel<F, G, CH, U, 2, RP, MINB, MASK>); break;
    case StepMode::Spmm: run(cheb_lean_kernel<F, G, CH, U, 3, RP, MINB, MASK>); break;
    case StepMode::SpmmAcc: run(cheb_lean_kernel<F, G, CH, U, 4, RP, MINB, MASK>); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

// Full-panel launch for qv vectors (qv a multiple of the chosen panel). Geometry
// measured on configs 1-2 (tools/tune_step.py): widest panel with one gathered
// row in flight per group and many resident warps.
template <class F, class RP>
void launch_full(adp_ctx* ctx, StepMode mode, const LArgs& k, int64_t qv, int64_t cap, const adp_csr* a) {
  if (qv % 128 == 0 && cap >= 128) return launch_lean<F, 32, 4, 1, RP, 4>(ctx, mode, k, qv);
  if (qv % 64 == 0 && cap >= 64) return launch_lean<F, 32, 2, 1, RP, 6>(ctx, mode, k, qv);
  if (qv % 32 == 0 && cap >= 32) return launch_lean<F, 32, 1, 1, RP, 8>(ctx, mode, k, qv);
  if (qv % 16 == 0) return launch_lean<F, 16, 1, 1, RP, 8>(ctx, mode, k, qv);
  if (qv % 8 == 0) return launch_lean<F, 8, 1, 1, RP, 8>(ctx, mode, k, qv);
  return launch_lean<F, 4, 1, 1, RP, 8>(ctx, mode, k, qv);  // qv % 4 == 0
}


// Masked geometry for a ragged tail of 5..127 vectors: quarter-warp groups up
// to 16 vectors, half-warp groups (two rows per warp in flight) up to 64,
// whole warps beyond (c1s solver widths: tools/tune_step.py --q).
template <class F, class RP>
void launch_masked_t(adp_ctx* ctx, StepMode mode, const LArgs& k, int64_t rem) {
  if (rem <= 16) return launch_lean<F, 8, 2, 1, RP, 8, true>(ctx, mode, k, rem);
  if (rem <= 32) return launch_lean<F, 16, 2, 1, RP, 6, true>(ctx, mode, k, rem);
  if (rem <= 48) return launch_lean<F, 16, 3, 1, RP, 4, true>(ctx, mode, k, rem);
  if (rem <= 64) return launch_lean<F, 16, 4, 1, RP, 4, true>(ctx, mode, k, rem);
  if (rem <= 96) return launch_lean<F, 32, 3, 1, RP, 4, true>(ctx, mode, k, rem);
  return launch_lean<F, 32, 4, 1, RP, 4, true>(ctx, mode, k, rem);
}

void launch_masked(adp_ctx* ctx, StepMode mode, const LArgs& k, int64_t rem, bool cplx, bool rp64) {
  if (cplx) {
    if (rp64) launch_masked_t<CplxL, int64_t>(ctx, mode, k, rem);
    else launch_masked_t<CplxL, int32_t>(ctx, mode, k, rem);
  } else {
    if (rp64) launch_masked_t<RealL, int64_t>(ctx, mode, k, rem);
    else launch_masked_t<RealL, int32_t>(ctx, mode, k, rem);
  }
}

}  // namespace

bool launch_step_lean(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  const adp_csr* a = s.a;
  const bool cplx = a->dtype == ADP_C128;
  const int epv = cplx ? 1 : 2;
  const int64_t qv = (s.q + epv - 1) / epv;
  if (qv < 4) return false;  // 1-3 vectors: the narrow-group row kernel
  LArgs k{};
  k.row_ptr = a->row_ptr;
  k.col = a->col_idx;
  k.val = a->values;
  k.g = static_cast<const char*>(s.gsrc);
  k.vin = static_cast<const char*>(s.vin);
  k.yin = static_cast<const char*>(s.yin);
  k.out = static_cast<char*>(s.out);
  k.wout = static_cast<char*>(s.wout);
  k.ldg_b = static_cast<uint32_t>((s.ld / epv) * 16);
  k.ldy_b = static_cast<uint32_t>((s.ld_y / epv) * 16);
  k.ldo_b = static_cast<uint32_t>((s.ld_out / epv) * 16);
  if (static_cast<int64_t>(k.ldg_b) != (s.ld / epv) * 16 || static_cast<int64_t>(k.ldo_b) != (s.ld_out / epv) * 16)
    return false;  // leading dimension beyond 32-bit byte offsets
  k.row_begin = s.row_begin;
  k.nrows = s.row_end - s.row_begin;
  k.goff = s.goff;
  k.g_rows = a->n_cols;
  k.s0 = s.s0;
  k.s1 = s.s1;
  k.s2 = s.s2;
  k.s3 = s.s3;
  k.n_push = s.n_push;
  for (int t = 0; t < s.n_push; ++t) k.push[t] = s.push[t];
  if (k.nrows >= (int64_t{1} << 30)) return false;
  // ragged widths: split into full-panel launches on column-offset pointers
  // panel cap (adp_ctx_set_panel): narrower panels shrink the L2 footprint of the
  // stencil's W reuse window at the cost of re-reading A once per panel
  const int64_t cap = ctx->panel_cols > 0 ? std::max<int64_t>(4, ctx->panel_cols / epv) : 128;
  int64_t done = 0;
  while (qv - done >= 4) {
    const int64_t rem = qv - done;
    int64_t take;
    const bool one_piece = rem == 4 || rem == 8 || rem == 16 || rem == 32 || rem == 64 || rem == 96;
    if (rem < 128 && rem > 4 && !one_piece && ctx->variant == 0 && cap >= 128) {
      // ragged tail of 5..127 vectors: ONE masked launch (a split into
      // power-of-two panels re-reads the operator and pays a launch per piece)
      LArgs kk = k;
      const uint32_t off = static_cast<uint32_t>(done * 16);
      kk.g += off;
      kk.vin = k.vin ? k.vin + off : nullptr;
      kk.yin = k.yin ? k.yin + off : nullptr;
      kk.out += off;
      kk.wout = k.wout ? k.wout + off : nullptr;
      for (int t = 0; t < kk.n_push; ++t) kk.push[t].dst += off;
      launch_masked(ctx, mode, kk, rem, cplx, a->rp64);
      done = qv;
      break;
    }
    if (rem >= 128 && cap >= 128) take = (rem / 128) * 128;
    else if (rem >= 64 && cap >= 64) take = (rem / 64) * 64;
    else if (rem >= 32 && cap >= 32) take = (rem / 32) * 32;
    else if (rem >= 64) take = 64;
    else if (rem >= 32) take = 32;
    else if (rem >= 16) take = 16;
    else if (rem >= 8) take = 8;
    else take = 4;
    LArgs kk = k;
    const uint32_t off = static_cast<uint32_t>(done * 16);
    kk.g += off;
    kk.vin = k.vin ? k.vin + off : nullptr;
    kk.yin = k.yin ? k.yin + off : nullptr;
    kk.out += off;
    kk.wout = k.wout ? k.wout + off : nullptr;
    for (int t = 0; t < kk.n_push; ++t) kk.push[t].dst += off;
    if (cplx) {
      if (a->rp64) launch_full<CplxL, int64_t>(ctx, mode, kk, take, cap, a);
      else launch_full<CplxL, int32_t>(ctx, mode, kk, take, cap, a);
    } else {
      if (a->rp64) launch_full<RealL, int64_t>(ctx, mode, kk, take, cap, a);
      else launch_full<RealL, int32_t>(ctx, mode, kk, take, cap, a);
    }
    done += take;
  }
  if (done < qv) {  // 1-3 remaining vectors: narrow-group row kernel on offset pointers
    StepArgs t = s;
    const int64_t off = done * 16;
    auto shift = [&](const void* ptr) -> void* {
      return ptr ? const_cast<char*>(static_cast<const char*>(ptr) + off) : nullptr;
    };
    t.gsrc = shift(s.gsrc);
    t.vin = shift(s.vin);
    t.yin = shift(s.yin);
    t.out = shift(s.out);
    t.wout = shift(s.wout);
    t.q = s.q - done * epv;
    PushTarget pt[kMaxPush];
    for (int i = 0; i < s.n_push; ++i) {
      pt[i] = s.push[i];
      pt[i].dst += off;
    }
    t.push = pt;
    launch_step(ctx, mode, t);
  }
  return true;
}

}  // namespace adp
