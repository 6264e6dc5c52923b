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

// ---- multi-row lean kernel ---------------------------------------------------------------
// cheb_lean_kernel's arithmetic and data movement, but each group walks RPW rows
// of its panel instead of one: the prologue (task decomposition, mbarrier init,
// cache policy) is paid once per RPW rows, the next row's row_ptr entry is the
// current row's end, and the next row's V / Y panels are bulk-copied into the
// group's (single) slot as soon as the epilogue has read it, so they land while
// the next row's gathers are in flight. STRD: the CTA's groups take rows
// rb + i*kGroups + grp (the 8 warps of a CTA work on 8 consecutive rows at any
// time, as in the one-row kernel, sharing x-neighbour gathers through L1);
// otherwise rows rb + grp*RPW + i (each warp re-gathers its previous row's
// neighbours). Rows are independent, so every bit of the result is unchanged.
template <class F, int G, int CH, int RPW, bool STRD, int MODE, class RP, int MINB, bool MASK = false>
__global__ void __launch_bounds__(kThreads, MINB) cheb_leanm_kernel(const LArgs p) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  constexpr int kGroups = kThreads / G;
  constexpr int kRowsPerCta = kGroups * RPW;
  constexpr uint32_t kPB = G * CH * 16u;
  extern __shared__ __align__(16) uint8_t smem[];

  const int grp = threadIdx.x / G, lane = threadIdx.x % G;
  const uint32_t gmask = G == 32 ? 0xffffffffu : (((1u << (G % 32)) - 1u) << ((threadIdx.x % 32) / G * G));
  const int32_t nrows = static_cast<int32_t>(p.nrows);
  const int32_t nblk = (nrows + kRowsPerCta - 1) / kRowsPerCta;
  const int32_t panel = static_cast<int32_t>(blockIdx.x) / nblk;  // CTA-uniform
  const int32_t rb = (static_cast<int32_t>(blockIdx.x) - panel * nblk) * kRowsPerCta;
  auto rel_row = [&](int i) -> int32_t { return STRD ? rb + i * kGroups + grp : rb + grp * RPW + i; };
  int32_t rel = rel_row(0);
  if (rel >= nrows) return;  // group-uniform
  const uint32_t poff = static_cast<uint32_t>(panel) * kPB;
  const uint32_t voff = poff + lane * 16u;
  const uint64_t pol = policy_evict_first(1.0f);

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + grp;
  double2* my = reinterpret_cast<double2*>(smem + ((kGroups * 8 + 15) / 16) * 16) + grp * (2 * G * CH);
  int64_t r = p.row_begin + rel;
  RP start = static_cast<RP>(ld_rp<RP>(p.row_ptr, r));
  RP end = static_cast<RP>(ld_rp<RP>(p.row_ptr, r + 1));
  pdl_wait_and_release();
  bool ok[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) ok[c] = !MASK || c * G + lane < p.valid;
  const uint32_t cpb = MASK ? static_cast<uint32_t>(p.valid) * 16u : kPB;
  if constexpr (kStep) {
    if (lane == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_arrive_expect_tx(bar, 2 * cpb);
      bulk_g2s_hint(my, p.vin + static_cast<uint64_t>(r) * p.ldg_b + poff, cpb, bar, pol);
      bulk_g2s_hint(my + G * CH, p.yin + static_cast<uint64_t>(r) * p.ldy_b + poff, cpb, bar, pol);
    }
  }
  const char* gb = p.g + voff;
  uint32_t phase = 0;
#pragma unroll 1
  for (int i = 0; i < RPW; ++i) {
    char* ob = p.out + static_cast<uint64_t>(r) * p.ldo_b + voff;
    double2 acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if constexpr (kSpmmAcc)
        acc[c] = ok[c] ? *reinterpret_cast<const double2*>(ob + G * 16 * c) : make_double2(0.0, 0.0);
      else
        acc[c] = make_double2(0.0, 0.0);
    }
    for (RP e = start; e < end; ++e) {
      const int cidx = __ldg(p.col + e);
      const auto v = F::load(p.val, static_cast<int64_t>(e));
      const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cidx)) * p.ldg_b);
      double2 w[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) w[c] = ok[c] ? __ldg(src + G * c) : make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        double2 wv = w[c];
        if constexpr (kFirst) wv = scale2(p.s2, wv);
        acc[c] = F::mac(acc[c], v, wv);
      }
    }
    // next row of this group (its row_ptr end is loaded before the epilogue's stores)
    const int32_t nrel = i + 1 < RPW ? rel_row(i + 1) : nrows;
    const bool more = nrel < nrows;
    if (more) {
      start = end;
      if (STRD) start = static_cast<RP>(ld_rp<RP>(p.row_ptr, p.row_begin + nrel));
      end = static_cast<RP>(ld_rp<RP>(p.row_ptr, p.row_begin + nrel + 1));
    }
    if constexpr (kStep) {
      __syncwarp(gmask);
      mbar_wait(bar, phase);
      phase ^= 1u;
    }
    const double2* own_src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(r + p.goff) * p.ldg_b);
    char* wb = kFirst ? p.wout + static_cast<uint64_t>(r) * p.ldo_b + voff : nullptr;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (!ok[c]) continue;
      double2 own = make_double2(0.0, 0.0);
      if constexpr (kNeedOwn) own = __ldg(own_src + G * c);
      double2 res;
      if constexpr (kStep) {
        const double2 vv = my[c * G + lane];
        const double2 yy = my[G * CH + c * G + lane];
        res = add2(sub2(add2(scale2(p.s0, acc[c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
      } else if constexpr (kFirst) {
        const double2 wn = scale2(p.s2, own);
        st_hint(wb + G * 16 * c, wn, pol);
        res = add2(scale2(p.s0, acc[c]), scale2(p.s1, wn));
      } else if constexpr (kDeg1) {
        res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[c]), scale2(p.s3, own))));
      } else {
        res = acc[c];
      }
      st_hint(ob + G * 16 * c, res, pol);
    }
    if (!more) break;  // group-uniform
    r = p.row_begin + nrel;
    if constexpr (kStep) {
      // the slot is free once every lane of the group has read it: refill it with the next row
      __syncwarp(gmask);
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive_expect_tx(bar, 2 * cpb);
        bulk_g2s_hint(my, p.vin + static_cast<uint64_t>(r) * p.ldg_b + poff, cpb, bar, pol);
        bulk_g2s_hint(my + G * CH, p.yin + static_cast<uint64_t>(r) * p.ldy_b + poff, cpb, bar, pol);
      }
    }
  }
}

template <class F, int G, int CH, int RPW, bool STRD, class RP, int MINB, bool MASK = false>
void launch_leanm(adp_ctx* ctx, StepMode mode, LArgs k, int64_t qv) {
  constexpr int kGroups = kThreads / G;
  k.n_panels = MASK ? 1 : qv / (G * CH);
  k.valid = static_cast<int32_t>(qv);
  const int64_t nblk = (k.nrows + kGroups * RPW - 1) / (kGroups * RPW);
  const int64_t grid64 = nblk * k.n_panels;
  if (grid64 >= (int64_t{1} << 31)) fail(ADP_ERR_DIMENSION, "cheb_leanm: too many CTAs");
  const int grid = static_cast<int>(grid64);
  const size_t smem = mode == StepMode::Step
                          ? static_cast<size_t>((kGroups * 8 + 15) / 16) * 16 + static_cast<size_t>(kGroups) * 2 * G * CH * 16
                          : 16;
  auto run = [&](auto kern) {
    if (smem > 48 * 1024)
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    launch_pdl(ctx, kern, dim3(grid), dim3(kThreads), smem, k);
  };
  switch (mode) {
    case StepMode::First: run(cheb_leanm_kernel<F, G, CH, RPW, STRD, 0, RP, MINB, MASK>); break;
    case StepMode::Step: run(cheb_leanm_kernel<F, G, CH, RPW, STRD, 1, RP, MINB, MASK>); break;
    case StepMode::Deg1: run(cheb_leanm_kernel<F, G, CH, RPW, STRD, 2, RP, MINB, MASK>); break;
    case StepMode::Spmm: run(cheb_leanm_kernel<F, G, CH, RPW, STRD, 3, RP, MINB, MASK>); break;
    case StepMode::SpmmAcc: run(cheb_leanm_kernel<F, G, CH, RPW, STRD, 4, RP, MINB, MASK>); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

// ---- row-block union kernel -----------------------------------------------------------
// A warp owns R consecutive rows of one panel and walks the UNION of their
// column sets in ascending order: every distinct W row panel is gathered once
// and fed to each of the R rows that contain it (the reference's column
// segments of a row block, tiled_matrix.hpp:78-91, done in registers). Each
// row still sees its own entries in ascending column order, so the arithmetic
// -- and every bit of the result -- is unchanged; the L1/L2 gather traffic
// drops by the operator's intra-block column overlap (27-point stencil, R = 4:
// 54 instead of 108 row-panel loads). Each row keeps its current and next
// (col, val) in registers so the union minimum never waits on a load.
template <class F, int CH, int R, int MODE, class RP, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) cheb_union_kernel(const LArgs p) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  constexpr int kWarps = kThreads / 32;
  constexpr uint32_t kPB = 32 * CH * 16u;
  constexpr int kNone = 0x7fffffff;
  using Val = typename F::Val;
  extern __shared__ __align__(16) uint8_t smem[];  // [8 mbarriers][warp][row][V, Y] panels

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int32_t nrows = static_cast<int32_t>(p.nrows);
  const int32_t nblk = (nrows + R - 1) / R;
  const int32_t task = static_cast<int32_t>(blockIdx.x) * kWarps + warp;
  if (task >= nblk * static_cast<int32_t>(p.n_panels)) return;
  const int32_t panel = task / nblk;
  const int32_t b = task - panel * nblk;
  const int64_t r0 = p.row_begin + static_cast<int64_t>(b) * R;
  const int rows = min(R, nrows - b * R);
  const uint32_t poff = static_cast<uint32_t>(panel) * kPB;
  const uint32_t voff = poff + lane * 16u;
  const uint64_t pol = policy_evict_first(1.0f);

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp;
  double2* my = reinterpret_cast<double2*>(smem + 128) + warp * (R * 2 * 32 * CH);
  if constexpr (kStep) {
    if (lane == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_arrive_expect_tx(bar, 2 * kPB * rows);
    }
    __syncwarp();
    if (lane < rows) {
      bulk_g2s_hint(my + lane * (2 * 32 * CH), p.vin + static_cast<uint64_t>(r0 + lane) * p.ldg_b + poff, kPB, bar, pol);
      bulk_g2s_hint(my + lane * (2 * 32 * CH) + 32 * CH, p.yin + static_cast<uint64_t>(r0 + lane) * p.ldy_b + poff, kPB,
                    bar, pol);
    }
  }
  const char* gb = p.g + voff;

  RP k[R], e[R];
  int c0[R], c1[R];
  Val v0[R], v1[R];
  double2 acc[R][CH];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    k[i] = 0;
    e[i] = 0;
    if (i < rows) {
      k[i] = static_cast<RP>(ld_rp<RP>(p.row_ptr, r0 + i));
      e[i] = static_cast<RP>(ld_rp<RP>(p.row_ptr, r0 + i + 1));
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if constexpr (kSpmmAcc)
        acc[i][c] = i < rows ? *reinterpret_cast<const double2*>(p.out + static_cast<uint64_t>(r0 + i) * p.ldo_b + voff + 512 * c)
                             : make_double2(0.0, 0.0);
      else
        acc[i][c] = make_double2(0.0, 0.0);
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    c0[i] = k[i] < e[i] ? __ldg(p.col + k[i]) : kNone;
    v0[i] = k[i] < e[i] ? F::load(p.val, k[i]) : Val{};
    c1[i] = k[i] + 1 < e[i] ? __ldg(p.col + k[i] + 1) : kNone;
    v1[i] = k[i] + 1 < e[i] ? F::load(p.val, k[i] + 1) : Val{};
  }
  while (true) {
    int cmin = c0[0];
#pragma unroll
    for (int i = 1; i < R; ++i) cmin = min(cmin, c0[i]);
    if (cmin == kNone) break;
    double2 w[CH];
    const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cmin)) * p.ldg_b);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      w[c] = __ldg(src + 32 * c);
      if constexpr (kFirst) w[c] = scale2(p.s2, w[c]);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (c0[i] == cmin) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[i][c] = F::mac(acc[i][c], v0[i], w[c]);
        ++k[i];
        c0[i] = c1[i];
        v0[i] = v1[i];
        c1[i] = k[i] + 1 < e[i] ? __ldg(p.col + k[i] + 1) : kNone;
        v1[i] = k[i] + 1 < e[i] ? F::load(p.val, k[i] + 1) : Val{};
      }
    }
  }
  if constexpr (kStep) {
    __syncwarp();
    mbar_wait(bar, 0);
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (i >= rows) break;
    const int64_t r = r0 + i;
    const double2* own_src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(r + p.goff) * p.ldg_b);
    char* ob = p.out + static_cast<uint64_t>(r) * p.ldo_b + voff;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double2 own = make_double2(0.0, 0.0);
      if constexpr (kNeedOwn) own = __ldg(own_src + 32 * c);
      double2 res;
      if constexpr (kStep) {
        const double2 vv = my[i * (2 * 32 * CH) + c * 32 + lane];
        const double2 yy = my[i * (2 * 32 * CH) + 32 * CH + c * 32 + lane];
        res = add2(sub2(add2(scale2(p.s0, acc[i][c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
      } else if constexpr (kFirst) {
        const double2 wn = scale2(p.s2, own);
        st_hint(p.wout + static_cast<uint64_t>(r) * p.ldo_b + voff + 512 * c, wn, pol);
        res = add2(scale2(p.s0, acc[i][c]), scale2(p.s1, wn));
      } else if constexpr (kDeg1) {
        res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[i][c]), scale2(p.s3, own))));
      } else {
        res = acc[i][c];
      }
      st_hint(ob + 512 * c, res, pol);
    }
  }
}

template <class F, int CH, int R, class RP, int MINB>
void launch_union(adp_ctx* ctx, StepMode mode, LArgs k, int64_t qv) {
  constexpr int kWarps = kThreads / 32;
  k.n_panels = qv / (32 * CH);
  const int64_t nblk = (k.nrows + R - 1) / R;
  const int64_t total = nblk * k.n_panels;
  if (total >= (int64_t{1} << 31)) fail(ADP_ERR_DIMENSION, "cheb_union: too many tasks");
  const int grid = static_cast<int>((total + kWarps - 1) / kWarps);
  const size_t smem = mode == StepMode::Step ? 128 + static_cast<size_t>(kWarps) * R * 2 * 32 * CH * 16 : 16;
  auto run = [&](auto kern) {
    if (smem > 48 * 1024)
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, kThreads, smem, ctx->stream>>>(k);
  };
  switch (mode) {
    case StepMode::First: run(cheb_union_kernel<F, CH, R, 0, RP, MINB>); break;
    case StepMode::Step: run(cheb_union_kernel<F, CH, R, 1, RP, MINB>); break;
    case StepMode::Deg1: run(cheb_union_kernel<F, CH, R, 2, RP, MINB>); break;
    case StepMode::Spmm: run(cheb_union_kernel<F, CH, R, 3, RP, MINB>); break;
    case StepMode::SpmmAcc: run(cheb_union_kernel<F, CH, R, 4, RP, MINB>); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

// ---- lean kernel with lane-parallel metadata ----------------------------------------------
// As cheb_lean_kernel (G = 32), but the row's (col, val) window is fetched with
// one coalesced load (lane k holds entry k) and broadcast by shuffles, so the W
// gathers depend on no memory load and U of them are issued back to back --
// removes the per-nonzero (col load -> W load) latency chain of long rows
// (27-point stencil, config 4).
template <class F, int CH, int U, int MODE, class RP, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) cheb_lean2_kernel(const LArgs p) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  constexpr int kWarps = kThreads / 32;
  constexpr uint32_t kPB = 32 * CH * 16u;
  using Val = typename F::Val;
  extern __shared__ __align__(16) uint8_t smem[];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int32_t nrows = static_cast<int32_t>(p.nrows);
  int32_t task = static_cast<int32_t>(blockIdx.x) * kWarps + warp;
  const bool live = task < nrows * static_cast<int32_t>(p.n_panels);
  if (!live) task = 0;  // no early return: keeps the warp provably converged at the shuffles
  const int32_t panel = task / nrows;
  const int64_t r = p.row_begin + (task - panel * nrows);
  const uint32_t poff = static_cast<uint32_t>(panel) * kPB;
  const uint32_t voff = poff + lane * 16u;
  const uint64_t pol = policy_evict_first(1.0f);

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp;
  double2* my = reinterpret_cast<double2*>(smem + 128) + warp * (2 * 32 * CH);
  if constexpr (kStep) {
    if (lane == 0 && live) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_arrive_expect_tx(bar, 2 * kPB);
      bulk_g2s_hint(my, p.vin + static_cast<uint64_t>(r) * p.ldg_b + poff, kPB, bar, pol);
      bulk_g2s_hint(my + 32 * CH, p.yin + static_cast<uint64_t>(r) * p.ldy_b + poff, kPB, bar, pol);
    }
  }
  char* ob = p.out + static_cast<uint64_t>(r) * p.ldo_b + voff;
  const char* gb = p.g + voff;
  double2 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if constexpr (kSpmmAcc)
      acc[c] = live ? *reinterpret_cast<const double2*>(ob + 512 * c) : make_double2(0.0, 0.0);
    else
      acc[c] = make_double2(0.0, 0.0);
  }
  const int64_t start = ld_rp<RP>(p.row_ptr, r);
  const int cnt_all = live ? static_cast<int>(ld_rp<RP>(p.row_ptr, r + 1) - start) : 0;
  for (int base = 0; base < cnt_all; base += 32) {
    const int cnt = min(32, cnt_all - base);
    int mc = 0;
    Val mv{};
    if (lane < cnt) {
      mc = __ldg(p.col + start + base + lane);
      mv = F::load(p.val, start + base + lane);
    }
    for (int k0 = 0; k0 < cnt; k0 += U) {
      double2 w[U][CH];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cidx = __shfl_sync(0xffffffffu, mc, (k0 + u) & 31);
        if (k0 + u < cnt) {
          const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cidx)) * p.ldg_b);
#pragma unroll
          for (int c = 0; c < CH; ++c) w[u][c] = __ldg(src + 32 * c);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        Val v;
        if constexpr (std::is_same<Val, double>::value) {
          v = __shfl_sync(0xffffffffu, mv, (k0 + u) & 31);
        } else {
          v.x = __shfl_sync(0xffffffffu, mv.x, (k0 + u) & 31);
          v.y = __shfl_sync(0xffffffffu, mv.y, (k0 + u) & 31);
        }
        if (k0 + u < cnt) {
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            double2 wv = w[u][c];
            if constexpr (kFirst) wv = scale2(p.s2, wv);
            acc[c] = F::mac(acc[c], v, wv);
          }
        }
      }
    }
  }
  if (!live) return;
  if constexpr (kStep) mbar_wait(bar, 0);
  const double2* own_src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(r + p.goff) * p.ldg_b);
  char* wb = kFirst ? p.wout + static_cast<uint64_t>(r) * p.ldo_b + voff : nullptr;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    double2 own = make_double2(0.0, 0.0);
    if constexpr (kNeedOwn) own = __ldg(own_src + 32 * c);
    double2 res;
    if constexpr (kStep) {
      const double2 vv = my[c * 32 + lane];
      const double2 yy = my[32 * CH + c * 32 + lane];
      res = add2(sub2(add2(scale2(p.s0, acc[c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
    } else if constexpr (kFirst) {
      const double2 wn = scale2(p.s2, own);
      st_hint(wb + 512 * c, wn, pol);
      res = add2(scale2(p.s0, acc[c]), scale2(p.s1, wn));
    } else if constexpr (kDeg1) {
      res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[c]), scale2(p.s3, own))));
    } else {
      res = acc[c];
    }
    st_hint(ob + 512 * c, res, pol);
  }
}

template <class F, int CH, int U, class RP, int MINB>
void launch_lean2(adp_ctx* ctx, StepMode mode, LArgs k, int64_t qv) {
  constexpr int kWarps = kThreads / 32;
  k.n_panels = qv / (32 * CH);
  const int64_t total = k.nrows * k.n_panels;
  if (total >= (int64_t{1} << 31)) fail(ADP_ERR_DIMENSION, "cheb_lean2: too many tasks");
  const int grid = static_cast<int>((total + kWarps - 1) / kWarps);
  const size_t smem = mode == StepMode::Step ? 128 + static_cast<size_t>(kWarps) * 2 * 32 * CH * 16 : 16;
  auto run = [&](auto kern) {
    if (smem > 48 * 1024)
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, kThreads, smem, ctx->stream>>>(k);
  };
  switch (mode) {
    case StepMode::First: run(cheb_lean2_kernel<F, CH, U, 0, RP, MINB>); break;
    case StepMode::Step: run(cheb_lean2_kernel<F, CH, U, 1, RP, MINB>); break;
    case StepMode::Deg1: run(cheb_lean2_kernel<F, CH, U, 2, RP, MINB>); break;
    case StepMode::Spmm: run(cheb_lean2_kernel<F, CH, U, 3, RP, MINB>); break;
    case StepMode::SpmmAcc: run(cheb_lean2_kernel<F, CH, U, 4, RP, MINB>); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

// ---- row-window kernel ----------------------------------------------------------------------
// A CTA of WARPS warps owns WARPS consecutive rows (one per warp) of one column
// panel. The gathered operand's rows [r0 - H, r0 + WARPS + H) -- the band every
// row of the block touches through its near-diagonal entries (the x-line of a
// stencil) and its own row -- are bulk-copied ONCE per CTA into shared memory;
// gathers whose column falls in that window read shared memory, the rest read
// global memory through L1 as in the lean kernel. Cuts the L2->SM gather
// traffic of a 7-point stencil from 7 to 4 + (WARPS+2H)/WARPS row panels per row
// and removes the own-row reload. Accumulation order per row is unchanged (CSR
// order), so results are bitwise the lean kernel's.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <class F, int CH, int WARPS, int H, int MODE, class RP, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) cheb_win_kernel(const LArgs p) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  constexpr uint32_t kPB = 32 * CH * 16u;
  constexpr int kWin = WARPS + 2 * H;
  using Val = typename F::Val;
  extern __shared__ __align__(16) uint8_t smem[];  // [2 mbarriers | pad][window rows][warp][V, Y]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int32_t nrows = static_cast<int32_t>(p.nrows);
  const int32_t nblk = (nrows + WARPS - 1) / WARPS;
  const int32_t panel = static_cast<int32_t>(blockIdx.x) / nblk;
  const int32_t b = static_cast<int32_t>(blockIdx.x) - panel * nblk;
  const int32_t rows = min(WARPS, nrows - b * WARPS);
  const int64_t r0 = p.row_begin + static_cast<int64_t>(b) * WARPS;  // first out row of the block
  const int64_t g0 = r0 + p.goff;                                     // its own row in the gathered operand
  const int64_t wlo = g0 - H > 0 ? g0 - H : 0;
  const int64_t whi = g0 + rows + H < p.g_rows ? g0 + rows + H : p.g_rows;
  const uint32_t wn = static_cast<uint32_t>(whi - wlo);
  const uint32_t poff = static_cast<uint32_t>(panel) * kPB;
  const uint32_t voff = poff + lane * 16u;

  uint64_t* wbar = reinterpret_cast<uint64_t*>(smem);
  uint64_t* vbar = wbar + 1;
  double2* win = reinterpret_cast<double2*>(smem + 128);
  double2* vy = win + kWin * 32 * CH;
  if (threadIdx.x == 0) {
    mbar_init(wbar, 1);
    mbar_init(vbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mbar_arrive_expect_tx(wbar, kPB * wn);
    if constexpr (kStep) mbar_arrive_expect_tx(vbar, 2 * kPB * static_cast<uint32_t>(rows));
  }
  __syncthreads();
  if (warp == 0) {
    const uint64_t pol = policy_evict_first(1.0f);
    for (uint32_t i = lane; i < wn; i += 32)  // WARPS + 2H may exceed 32
      bulk_g2s(win + i * 32 * CH, p.g + static_cast<uint64_t>(wlo + i) * p.ldg_b + poff, kPB, wbar);
    if constexpr (kStep) {
      if (lane < rows) {
        bulk_g2s_hint(vy + lane * 2 * 32 * CH, p.vin + static_cast<uint64_t>(r0 + lane) * p.ldg_b + poff, kPB, vbar, pol);
        bulk_g2s_hint(vy + lane * 2 * 32 * CH + 32 * CH, p.yin + static_cast<uint64_t>(r0 + lane) * p.ldy_b + poff, kPB,
                      vbar, pol);
      }
    }
  }
  if (warp >= rows) return;
  const uint64_t pol = policy_evict_first(1.0f);
  const int64_t r = r0 + warp;
  char* ob = p.out + static_cast<uint64_t>(r) * p.ldo_b + voff;
  const char* gb = p.g + voff;
  double2 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if constexpr (kSpmmAcc)
      acc[c] = *reinterpret_cast<const double2*>(ob + 512 * c);
    else
      acc[c] = make_double2(0.0, 0.0);
  }
  bool ready = false;
  const RP start = static_cast<RP>(ld_rp<RP>(p.row_ptr, r));
  const RP end = static_cast<RP>(ld_rp<RP>(p.row_ptr, r + 1));
  for (RP e = start; e < end; ++e) {
    const int cidx = __ldg(p.col + e);
    const Val v = F::load(p.val, static_cast<int64_t>(e));
    const uint32_t rel = static_cast<uint32_t>(cidx - static_cast<int32_t>(wlo));
    double2 w[CH];
    if (rel < wn) {
      if (!ready) {
        mbar_wait(wbar, 0);
        ready = true;
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) w[c] = win[rel * (32 * CH) + c * 32 + lane];
    } else {
      const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cidx)) * p.ldg_b);
#pragma unroll
      for (int c = 0; c < CH; ++c) w[c] = __ldg(src + 32 * c);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double2 wv = w[c];
      if constexpr (kFirst) wv = scale2(p.s2, wv);
      acc[c] = F::mac(acc[c], v, wv);
    }
  }
  if (!ready) mbar_wait(wbar, 0);  // also: no CTA exit with bulk copies in flight
  if constexpr (kStep) mbar_wait(vbar, 0);
  const uint32_t own_rel = static_cast<uint32_t>(g0 + warp - wlo);
  char* wb = kFirst ? p.wout + static_cast<uint64_t>(r) * p.ldo_b + voff : nullptr;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    double2 own = make_double2(0.0, 0.0);
    if constexpr (kNeedOwn) own = win[own_rel * (32 * CH) + c * 32 + lane];
    double2 res;
    if constexpr (kStep) {
      const double2 vv = vy[warp * 2 * 32 * CH + c * 32 + lane];
      const double2 yy = vy[warp * 2 * 32 * CH + 32 * CH + c * 32 + lane];
      res = add2(sub2(add2(scale2(p.s0, acc[c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
    } else if constexpr (kFirst) {
      const double2 wn2 = scale2(p.s2, own);
      st_hint(wb + 512 * c, wn2, pol);
      res = add2(scale2(p.s0, acc[c]), scale2(p.s1, wn2));
    } else if constexpr (kDeg1) {
      res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[c]), scale2(p.s3, own))));
    } else {
      res = acc[c];
    }
    st_hint(ob + 512 * c, res, pol);
  }
}

template <class F, int CH, int WARPS, int H, class RP, int MINB>
void launch_win(adp_ctx* ctx, StepMode mode, LArgs k, int64_t qv) {
  k.n_panels = qv / (32 * CH);
  const int64_t nblk = (k.nrows + WARPS - 1) / WARPS;
  const int64_t total = nblk * k.n_panels;
  if (total >= (int64_t{1} << 31)) fail(ADP_ERR_DIMENSION, "cheb_win: too many blocks");
  constexpr size_t kWinBytes = static_cast<size_t>(WARPS + 2 * H) * 32 * CH * 16;
  const size_t smem = 128 + kWinBytes + (mode == StepMode::Step ? static_cast<size_t>(WARPS) * 2 * 32 * CH * 16 : 0);
  auto run = [&](auto kern) {
    if (smem > 48 * 1024)
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<static_cast<int>(total), WARPS * 32, smem, ctx->stream>>>(k);
  };
  switch (mode) {
    case StepMode::First: run(cheb_win_kernel<F, CH, WARPS, H, 0, RP, MINB>); break;
    case StepMode::Step: run(cheb_win_kernel<F, CH, WARPS, H, 1, RP, MINB>); break;
    case StepMode::Deg1: run(cheb_win_kernel<F, CH, WARPS, H, 2, RP, MINB>); break;
    case StepMode::Spmm: run(cheb_win_kernel<F, CH, WARPS, H, 3, RP, MINB>); break;
    case StepMode::SpmmAcc: run(cheb_win_kernel<F, CH, WARPS, H, 4, RP, MINB>); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

// ---- column-segment kernel (MaSpMM row blocks) ------------------------------------------
// A warp owns an R-row block of one panel and walks the block's precomputed
// distinct columns (segments.cpp): each W row panel is loaded ONCE and applied,
// from registers, to every row of the block whose bit is set in the segment's
// mask. Unlike the union kernel the walk has no loop-carried dependency (the
// segment list is data), so U segments are loaded ahead. Per row the products
// still accumulate in ascending column order: bitwise the reference's.
struct SArgs {
  LArgs l;
  const int64_t* blk_ptr;
  const int32_t* seg_col;
  const uint32_t* seg_mask;
  const void* seg_val;
};

template <class F, int CH, int R, int U, int MODE, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) cheb_seg_kernel(const SArgs sa) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  constexpr int kWarps = kThreads / 32;
  constexpr uint32_t kPB = 32 * CH * 16u;
  using Val = typename F::Val;
  const LArgs& p = sa.l;
  extern __shared__ __align__(16) uint8_t smem[];  // [8 mbarriers][warp][row][V, Y] panels

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int32_t nrows = static_cast<int32_t>(p.nrows);
  const int32_t nblk = (nrows + R - 1) / R;
  const int32_t task = static_cast<int32_t>(blockIdx.x) * kWarps + warp;
  if (task >= nblk * static_cast<int32_t>(p.n_panels)) return;
  const int32_t panel = task / nblk;
  const int32_t b = task - panel * nblk;
  const int64_t r0 = static_cast<int64_t>(b) * R;  // segments cover the whole operator (row_begin == 0)
  const int rows = min(R, nrows - b * R);
  const uint32_t poff = static_cast<uint32_t>(panel) * kPB;
  const uint32_t voff = poff + lane * 16u;
  const uint64_t pol = policy_evict_first(1.0f);

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp;
  double2* my = reinterpret_cast<double2*>(smem + 128) + warp * (R * 2 * 32 * CH);
  if constexpr (kStep) {
    if (lane == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_arrive_expect_tx(bar, 2 * kPB * rows);
    }
    __syncwarp();
    if (lane < rows) {
      bulk_g2s_hint(my + lane * (2 * 32 * CH), p.vin + static_cast<uint64_t>(r0 + lane) * p.ldg_b + poff, kPB, bar, pol);
      bulk_g2s_hint(my + lane * (2 * 32 * CH) + 32 * CH, p.yin + static_cast<uint64_t>(r0 + lane) * p.ldy_b + poff, kPB,
                    bar, pol);
    }
  }
  const char* gb = p.g + voff;
  double2 acc[R][CH];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if constexpr (kSpmmAcc)
        acc[i][c] = i < rows ? *reinterpret_cast<const double2*>(p.out + static_cast<uint64_t>(r0 + i) * p.ldo_b + voff + 512 * c)
                             : make_double2(0.0, 0.0);
      else
        acc[i][c] = make_double2(0.0, 0.0);
    }
  const int64_t s0 = __ldg(sa.blk_ptr + b), s1 = __ldg(sa.blk_ptr + b + 1);
  for (int64_t s = s0; s < s1; s += U) {
    int col[U];
    uint32_t msk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      col[u] = 0;
      msk[u] = 0;
      if (s + u < s1) {
        col[u] = __ldg(sa.seg_col + s + u);
        msk[u] = __ldg(sa.seg_mask + s + u);
      }
    }
    double2 w[U][CH];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (s + u < s1) {
        const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(col[u])) * p.ldg_b);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          w[u][c] = __ldg(src + 32 * c);
          if constexpr (kFirst) w[u][c] = scale2(p.s2, w[u][c]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if ((msk[u] >> i) & 1u) {
          const Val v = F::load(sa.seg_val, (s + u) * R + i);
#pragma unroll
          for (int c = 0; c < CH; ++c) acc[i][c] = F::mac(acc[i][c], v, w[u][c]);
        }
      }
    }
  }
  if constexpr (kStep) {
    __syncwarp();
    mbar_wait(bar, 0);
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (i >= rows) break;
    const int64_t r = r0 + i;
    const double2* own_src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(r + p.goff) * p.ldg_b);
    char* ob = p.out + static_cast<uint64_t>(r) * p.ldo_b + voff;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double2 own = make_double2(0.0, 0.0);
      if constexpr (kNeedOwn) own = __ldg(own_src + 32 * c);
      double2 res;
      if constexpr (kStep) {
        const double2 vv = my[i * (2 * 32 * CH) + c * 32 + lane];
        const double2 yy = my[i * (2 * 32 * CH) + 32 * CH + c * 32 + lane];
        res = add2(sub2(add2(scale2(p.s0, acc[i][c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
      } else if constexpr (kFirst) {
        const double2 wn = scale2(p.s2, own);
        st_hint(p.wout + static_cast<uint64_t>(r) * p.ldo_b + voff + 512 * c, wn, pol);
        res = add2(scale2(p.s0, acc[i][c]), scale2(p.s1, wn));
      } else if constexpr (kDeg1) {
        res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[i][c]), scale2(p.s3, own))));
      } else {
        res = acc[i][c];
      }
      st_hint(ob + 512 * c, res, pol);
    }
  }
}

template <class F, int CH, int R, int U, int MINB>
bool launch_seg(adp_ctx* ctx, StepMode mode, const LArgs& k, int64_t qv, const adp_csr* a) {
  if (k.row_begin != 0 || k.nrows != a->n_rows) return false;  // segments cover whole operators
  const Segments* sg = get_segments(const_cast<adp_csr*>(a), R);
  constexpr int kWarps = kThreads / 32;
  SArgs sa{};
  sa.l = k;
  sa.l.n_panels = qv / (32 * CH);
  sa.blk_ptr = static_cast<const int64_t*>(sg->d_blk_ptr);
  sa.seg_col = static_cast<const int32_t*>(sg->d_col);
  sa.seg_mask = static_cast<const uint32_t*>(sg->d_mask);
  sa.seg_val = sg->d_val;
  const int64_t total = sg->n_blocks * sa.l.n_panels;
  if (total >= (int64_t{1} << 31)) return false;
  const int grid = static_cast<int>((total + kWarps - 1) / kWarps);
  const size_t smem = mode == StepMode::Step ? 128 + static_cast<size_t>(kWarps) * R * 2 * 32 * CH * 16 : 16;
  auto run = [&](auto kern) {
    if (smem > 48 * 1024)
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, kThreads, smem, ctx->stream>>>(sa);
  };
  switch (mode) {
    case StepMode::First: run(cheb_seg_kernel<F, CH, R, U, 0, MINB>); break;
    case StepMode::Step: run(cheb_seg_kernel<F, CH, R, U, 1, MINB>); break;
    case StepMode::Deg1: run(cheb_seg_kernel<F, CH, R, U, 2, MINB>); break;
    case StepMode::Spmm: run(cheb_seg_kernel<F, CH, R, U, 3, MINB>); break;
    case StepMode::SpmmAcc: run(cheb_seg_kernel<F, CH, R, U, 4, MINB>); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
  return true;
}

// Full-panel launch for qv vectors (qv a multiple of the chosen panel). Geometry
// measured on configs 1-2 (tools/tune_step.py): widest panel with one gathered
// row in flight per group and many resident warps.
template <class F, class RP>
void launch_full(adp_ctx* ctx, StepMode mode, const LArgs& k, int64_t qv, int64_t cap, const adp_csr* a) {
  switch (ctx->variant) {  // row-block union kernel (tuning variants 21-24)
    case 21: if (qv % 64 == 0) return launch_union<F, 2, 4, RP, 3>(ctx, mode, k, qv); break;
    case 22: if (qv % 128 == 0) return launch_union<F, 4, 2, RP, 2>(ctx, mode, k, qv); break;
    case 23: if (qv % 64 == 0) return launch_union<F, 2, 2, RP, 4>(ctx, mode, k, qv); break;
    case 24: if (qv % 32 == 0) return launch_union<F, 1, 4, RP, 4>(ctx, mode, k, qv); break;
    // deeper gather batches for long rows (tuning variants 31-33)
    case 31: if (qv % 32 == 0) return launch_lean<F, 32, 1, 8, RP, 4>(ctx, mode, k, qv); break;
    case 32: if (qv % 64 == 0) return launch_lean<F, 32, 2, 4, RP, 3>(ctx, mode, k, qv); break;
    case 33: if (qv % 128 == 0) return launch_lean<F, 32, 4, 4, RP, 2>(ctx, mode, k, qv); break;
    // column-segment (MaSpMM row-block) kernel (tuning variants 41-46)
    case 41: if (qv % 64 == 0 && launch_seg<F, 2, 4, 2, 2>(ctx, mode, k, qv, a)) return; break;
    case 42: if (qv % 128 == 0 && launch_seg<F, 4, 2, 2, 2>(ctx, mode, k, qv, a)) return; break;
    case 43: if (qv % 32 == 0 && launch_seg<F, 1, 8, 2, 2>(ctx, mode, k, qv, a)) return; break;
    case 44: if (qv % 64 == 0 && launch_seg<F, 2, 2, 4, 3>(ctx, mode, k, qv, a)) return; break;
    case 45: if (qv % 32 == 0 && launch_seg<F, 1, 4, 4, 4>(ctx, mode, k, qv, a)) return; break;
    case 46: if (qv % 128 == 0 && launch_seg<F, 4, 4, 1, 1>(ctx, mode, k, qv, a)) return; break;
    case 47: if (qv % 128 == 0 && launch_seg<F, 4, 4, 1, 2>(ctx, mode, k, qv, a)) return; break;
    case 48: if (qv % 64 == 0 && launch_seg<F, 2, 4, 2, 3>(ctx, mode, k, qv, a)) return; break;
    case 49: if (qv % 64 == 0 && launch_seg<F, 2, 4, 1, 4>(ctx, mode, k, qv, a)) return; break;
    case 40: if (qv % 128 == 0 && launch_seg<F, 4, 3, 1, 2>(ctx, mode, k, qv, a)) return; break;
    // lane-parallel metadata (tuning variants 51-56)
    case 51: if (qv % 128 == 0) return launch_lean2<F, 4, 2, RP, 2>(ctx, mode, k, qv); break;
    case 52: if (qv % 128 == 0) return launch_lean2<F, 4, 4, RP, 2>(ctx, mode, k, qv); break;
    case 53: if (qv % 64 == 0) return launch_lean2<F, 2, 4, RP, 3>(ctx, mode, k, qv); break;
    case 54: if (qv % 64 == 0) return launch_lean2<F, 2, 8, RP, 2>(ctx, mode, k, qv); break;
    case 55: if (qv % 32 == 0) return launch_lean2<F, 1, 8, RP, 4>(ctx, mode, k, qv); break;
    case 56: if (qv % 128 == 0) return launch_lean2<F, 4, 1, RP, 4>(ctx, mode, k, qv); break;
    // row-window kernel (tuning variants 61-66)
    case 61: if (qv % 128 == 0) return launch_win<F, 4, 8, 1, RP, 4>(ctx, mode, k, qv); break;
    case 62: if (qv % 128 == 0) return launch_win<F, 4, 16, 1, RP, 2>(ctx, mode, k, qv); break;
    case 63: if (qv % 64 == 0) return launch_win<F, 2, 8, 1, RP, 6>(ctx, mode, k, qv); break;
    case 64: if (qv % 128 == 0) return launch_win<F, 4, 32, 1, RP, 1>(ctx, mode, k, qv); break;
    case 65: if (qv % 64 == 0) return launch_win<F, 2, 16, 1, RP, 3>(ctx, mode, k, qv); break;
    case 66: if (qv % 128 == 0) return launch_win<F, 4, 4, 1, RP, 8>(ctx, mode, k, qv); break;
    // multi-row lean kernel (tuning variants 101-108)
    case 101: if (qv % 128 == 0) return launch_leanm<F, 32, 4, 2, true, RP, 4>(ctx, mode, k, qv); break;
    case 102: if (qv % 128 == 0) return launch_leanm<F, 32, 4, 4, true, RP, 4>(ctx, mode, k, qv); break;
    case 103: if (qv % 128 == 0) return launch_leanm<F, 32, 4, 8, true, RP, 4>(ctx, mode, k, qv); break;
    case 104: if (qv % 128 == 0) return launch_leanm<F, 32, 4, 2, false, RP, 4>(ctx, mode, k, qv); break;
    case 105: if (qv % 128 == 0) return launch_leanm<F, 32, 4, 4, false, RP, 4>(ctx, mode, k, qv); break;
    case 106: if (qv % 128 == 0) return launch_leanm<F, 32, 4, 8, false, RP, 4>(ctx, mode, k, qv); break;
    case 107: if (qv % 64 == 0) return launch_leanm<F, 32, 2, 4, true, RP, 6>(ctx, mode, k, qv); break;
    case 108: if (qv % 64 == 0) return launch_leanm<F, 32, 2, 4, false, RP, 6>(ctx, mode, k, qv); break;
    default: break;
  }
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
