// Persistent, software-pipelined fused Clenshaw step (sm_100a) -- the default
// kernel for blocks of >= 64 fp64 columns (>= 32 complex).
//
// One warp owns a (row, column panel) task at a time; lane l holds CH 16-byte
// vectors of the panel, so each gathered W row panel is CH fully coalesced
// 512-byte warp loads. Warps are persistent (grid = SMs x resident blocks) and
// walk task chunks in row-ascending, panel-major order, which keeps the active
// rows of the whole GPU inside a narrow window -- the stencil's W reuse is then
// served by L2 (measured: DRAM bytes within 6% of the algorithmic minimum).
//
// The per-row dependency chain (row_ptr -> col/val -> W gathers -> epilogue
// operands) is broken by pipelining across the warp's task sequence:
//   iteration t: issue row_ptr loads of task t+2,
//                issue col/val loads of task t+1 (its row_ptr arrived at t-1),
//                cp.async V/Y panels of task t+1 into a per-warp smem ring,
//                gather W for task t (its col/val arrived at t-1), reduce,
//                wait for task t's V/Y (cp.async.wait_group 1), store.
// so every load is issued one or two tasks before it is consumed.
//
// Arithmetic: unfused __dmul_rn/__dadd_rn in CSR (ascending-column) order and
// the reference's expression order -- bitwise identical to the reference
// (proj/include/adapoly/tiled_matrix.hpp:205, proj/src/cheb_filter.cpp:162-177).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "adp_internal.hpp"

namespace adp {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int64_t kChunk = 8;  // consecutive tasks per warp chunk

struct RArgs {
  const void* row_ptr;
  const int32_t* col;
  const void* val;
  const double2* g;
  const double2* vin;
  const double2* yin;
  double2* out;
  double2* wout;
  int64_t ldv, ldyv, ldo, qv, row_begin, nrows, n_panels, goff;
  double s0, s1, s2, s3;
  float pol_frac;  // 1.0: L2 evict-first fraction, a runtime operand so ptxas cannot fold the policy
};

struct RealV {
  using Val = double;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double*>(p) + k); }
  static __device__ __forceinline__ Val shfl(Val v, int src) { return __shfl_sync(0xffffffffu, v, src); }
  static __device__ __forceinline__ Val zero() { return 0.0; }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};
struct CplxV {
  using Val = double2;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double2*>(p) + k); }
  static __device__ __forceinline__ Val shfl(Val v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
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
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first_rt(float frac) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, %1;\n" : "=l"(pol) : "f"(frac));
  return pol;
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
template <class RP>
__device__ __forceinline__ int64_t ld_rp(const void* p, int64_t i) {
  return static_cast<int64_t>(__ldg(static_cast<const RP*>(p) + i));
}

// A task = (panel, row). Tasks are grouped into chunks of kChunk consecutive
// rows of one panel; chunk c goes to warp c mod n_warps (row-ascending fronts).
struct Task {
  int32_t row;    // -1 = none
  int32_t panel;
};

struct TaskWalker {
  int32_t chunk;       // current chunk id
  int32_t i;           // index inside the chunk
  int32_t n_warps, chunks_per_panel, n_chunks;
  int32_t nrows;
  __device__ __forceinline__ Task current() const {
    if (chunk >= n_chunks) return Task{-1, 0};
    const int32_t panel = chunk / chunks_per_panel;  // 32-bit: one cheap division per task
    const int32_t row = (chunk - panel * chunks_per_panel) * static_cast<int32_t>(kChunk) + i;
    return Task{row, panel};
  }
  __device__ __forceinline__ void advance() {
    const Task t = current();
    if (t.row < 0) return;
    if (i + 1 < kChunk && t.row + 1 < nrows) {
      ++i;
    } else {
      chunk += n_warps;
      i = 0;
    }
  }
};

template <class F, int CH, int U, int MODE, class RP, int MINB, bool FULL>
__global__ void __launch_bounds__(kThreads, MINB) cheb_row_kernel(const RArgs p) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  using Val = typename F::Val;

  // per-warp ring (dynamic smem): [2 buffers][V, Y][CH][32 lanes] 16-byte vectors
  extern __shared__ double2 ring[];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t n_warps = static_cast<int64_t>(gridDim.x) * kWarps;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  const uint64_t pol = policy_evict_first();
  TaskWalker walk{static_cast<int32_t>(gw), 0, static_cast<int32_t>(n_warps),
                  static_cast<int32_t>((p.nrows + kChunk - 1) / kChunk), 0, static_cast<int32_t>(p.nrows)};
  walk.n_chunks = walk.chunks_per_panel * static_cast<int32_t>(p.n_panels);
  double2* my_ring = ring + warp * (2 * 2 * CH * 32);

  auto vec_ok = [&](int32_t panel, int c) {
    return FULL || static_cast<int64_t>(panel) * (32 * CH) + lane + 32 * c < p.qv;
  };
  auto issue_vy = [&](const Task& t, int b) {
    if constexpr (kStep) {
      if (t.row >= 0) {
        const int64_t r = p.row_begin + t.row;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          if (vec_ok(t.panel, c)) {
            const int64_t v = static_cast<int64_t>(t.panel) * (32 * CH) + lane + 32 * c;
            cp_async16_hint(&my_ring[((b * 2 + 0) * CH + c) * 32 + lane], p.vin + r * p.ldv + v, pol);
            cp_async16_hint(&my_ring[((b * 2 + 1) * CH + c) * 32 + lane], p.yin + r * p.ldyv + v, pol);
          }
        }
      }
      cp_async_commit();
    }
  };

  // prologue: task 0 (row_ptr, col/val, V/Y) and task 1 (row_ptr)
  Task t0 = walk.current();
  if (t0.row < 0) return;
  walk.advance();
  Task t1 = walk.current();
  walk.advance();
  RP s0 = 0, e0 = 0, s1 = 0, e1 = 0;
  s0 = static_cast<RP>(ld_rp<RP>(p.row_ptr, p.row_begin + t0.row));
  e0 = static_cast<RP>(ld_rp<RP>(p.row_ptr, p.row_begin + t0.row + 1));
  if (t1.row >= 0) {
    s1 = static_cast<RP>(ld_rp<RP>(p.row_ptr, p.row_begin + t1.row));
    e1 = static_cast<RP>(ld_rp<RP>(p.row_ptr, p.row_begin + t1.row + 1));
  }
  int col0 = 0;
  Val val0 = F::zero();
  if (lane < e0 - s0) {
    col0 = __ldg(p.col + s0 + lane);
    val0 = F::load(p.val, static_cast<int64_t>(s0) + lane);
  }
  int buf = 0;
  issue_vy(t0, 0);

  while (t0.row >= 0) {
    // ---- prefetch: row_ptr of task +2; col/val and V/Y of task +1
    const Task t2 = walk.current();
    walk.advance();
    RP s2 = 0, e2 = 0;
    if (t2.row >= 0) {
      s2 = static_cast<RP>(ld_rp<RP>(p.row_ptr, p.row_begin + t2.row));
      e2 = static_cast<RP>(ld_rp<RP>(p.row_ptr, p.row_begin + t2.row + 1));
    }
    int col1 = 0;
    Val val1 = F::zero();
    if (t1.row >= 0 && lane < e1 - s1) {
      col1 = __ldg(p.col + s1 + lane);
      val1 = F::load(p.val, static_cast<int64_t>(s1) + lane);
    }
    issue_vy(t1, buf ^ 1);

    // ---- task 0: gather W rows in CSR order and reduce
    const int64_t r = p.row_begin + t0.row;
    const int64_t vbase = static_cast<int64_t>(t0.panel) * (32 * CH) + lane;
    bool ok[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) ok[c] = vec_ok(t0.panel, c);
    double2 acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if constexpr (kSpmmAcc)
        acc[c] = ok[c] ? p.out[r * p.ldo + vbase + 32 * c] : make_double2(0.0, 0.0);
      else
        acc[c] = make_double2(0.0, 0.0);
    }
    const int cnt_all = static_cast<int>(e0 - s0);
    for (int base = 0; base < cnt_all; base += 32) {
      int mc = col0;
      Val mv = val0;
      if (base > 0) {  // rows longer than 32 nonzeros: next metadata window
        mc = 0;
        mv = F::zero();
        if (lane < cnt_all - base) {
          mc = __ldg(p.col + s0 + base + lane);
          mv = F::load(p.val, static_cast<int64_t>(s0) + base + lane);
        }
      }
      const int cnt = min(32, cnt_all - base);
      for (int k0 = 0; k0 < cnt; k0 += U) {
        double2 w[U][CH];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int cidx = __shfl_sync(0xffffffffu, mc, (k0 + u) & 31);
          if (k0 + u < cnt) {
            const double2* src = p.g + static_cast<int64_t>(cidx) * p.ldv + vbase;
#pragma unroll
            for (int c = 0; c < CH; ++c)
              if (ok[c]) w[u][c] = __ldg(src + 32 * c);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const Val v = F::shfl(mv, (k0 + u) & 31);
          if (k0 + u < cnt) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              if (!ok[c]) continue;
              double2 wv = w[u][c];
              if constexpr (kFirst) wv = scale2(p.s2, wv);
              acc[c] = F::mac(acc[c], v, wv);
            }
          }
        }
      }
    }

    // ---- epilogue of task 0 (own row: an L1 hit -- it was just gathered as the diagonal)
    if constexpr (kStep) cp_async_wait<1>();
    const double2* own_src = p.g + (r + p.goff) * p.ldv + vbase;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (!ok[c]) continue;
      double2 own = make_double2(0.0, 0.0);
      if constexpr (kNeedOwn) own = __ldg(own_src + 32 * c);
      double2* dst = p.out + r * p.ldo + vbase + 32 * c;
      double2 res;
      if constexpr (kStep) {
        const double2 vv = my_ring[((buf * 2 + 0) * CH + c) * 32 + lane];
        const double2 yy = my_ring[((buf * 2 + 1) * CH + c) * 32 + lane];
        res = add2(sub2(add2(scale2(p.s0, acc[c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
      } else if constexpr (kFirst) {
        const double2 wn = scale2(p.s2, own);
        st_hint(p.wout + r * p.ldo + vbase + 32 * c, wn, pol);
        res = add2(scale2(p.s0, acc[c]), scale2(p.s1, wn));
      } else if constexpr (kDeg1) {
        res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[c]), scale2(p.s3, own))));
      } else {
        res = acc[c];
      }
      st_hint(dst, res, pol);
    }

    // ---- rotate the pipeline
    t0 = t1;
    s0 = s1;
    e0 = e1;
    col0 = col1;
    val0 = val1;
    t1 = t2;
    s1 = s2;
    e1 = e2;
    buf ^= 1;
  }
  if constexpr (kStep) cp_async_wait<0>();
}

template <class F, int CH, int U, class RP, int MINB, bool FULL>
void launch_row(adp_ctx* ctx, StepMode mode, const RArgs& k) {
  const int64_t total = k.nrows * k.n_panels;
  const int64_t chunks = (total + kChunk - 1) / kChunk;
  const int64_t want_blocks = (chunks + kWarps - 1) / kWarps;
  const int grid = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(want_blocks, static_cast<int64_t>(ctx->sm_count) * MINB)));
  const size_t smem = mode == StepMode::Step ? static_cast<size_t>(kWarps) * 2 * 2 * CH * 32 * 16 : 16;
  auto run = [&](auto kern) {
    const cudaError_t prior = cudaGetLastError();
    if (prior != cudaSuccess) fail(ADP_ERR_CUDA, std::string("pending CUDA error before cheb_row launch: ") +
                                                     cudaGetErrorString(prior));
    if (smem > 48 * 1024) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
      if (e != cudaSuccess)
        fail(ADP_ERR_CUDA, std::string("cheb_row: cudaFuncSetAttribute(smem=") + std::to_string(smem) +
                               "): " + cudaGetErrorString(e));
    }
    kern<<<grid, kThreads, smem, ctx->stream>>>(k);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
      fail(ADP_ERR_CUDA, std::string("cheb_row launch (grid ") + std::to_string(grid) + ", smem " +
                             std::to_string(smem) + ", CH " + std::to_string(CH) + "): " + cudaGetErrorString(e));
  };
  switch (mode) {
    case StepMode::First: run(cheb_row_kernel<F, CH, U, 0, RP, MINB, FULL>); break;
    case StepMode::Step: run(cheb_row_kernel<F, CH, U, 1, RP, MINB, FULL>); break;
    case StepMode::Deg1: run(cheb_row_kernel<F, CH, U, 2, RP, MINB, FULL>); break;
    case StepMode::Spmm: run(cheb_row_kernel<F, CH, U, 3, RP, MINB, FULL>); break;
    case StepMode::SpmmAcc: run(cheb_row_kernel<F, CH, U, 4, RP, MINB, FULL>); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

template <class F, class RP, int CH, int U, int MINB>
void launch_ch(adp_ctx* ctx, StepMode mode, RArgs k) {
  k.n_panels = (k.qv + 32 * CH - 1) / (32 * CH);
  if (k.qv % (32 * CH) == 0)
    launch_row<F, CH, U, RP, MINB, true>(ctx, mode, k);
  else
    launch_row<F, CH, U, RP, MINB, false>(ctx, mode, k);
}


template <class F, class RP>
void dispatch_row(adp_ctx* ctx, StepMode mode, const RArgs& k, int pipe_variant) {
  // tuning variants (adp_ctx_set_tuning 11..15) of the persistent pipelined kernel
  switch (pipe_variant) {
    case 1: return launch_ch<F, RP, 4, 4, 2>(ctx, mode, k);
    case 2: return launch_ch<F, RP, 2, 8, 2>(ctx, mode, k);
    case 3: return launch_ch<F, RP, 2, 4, 3>(ctx, mode, k);
    case 4: return launch_ch<F, RP, 3, 4, 2>(ctx, mode, k);
    default: return launch_ch<F, RP, 2, 4, 3>(ctx, mode, k);
  }
}

}  // namespace

bool launch_step_row(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  const adp_csr* a = s.a;
  const bool cplx = a->dtype == ADP_C128;
  const int epv = cplx ? 1 : 2;
  const int64_t qv = (s.q + epv - 1) / epv;
  if (qv < 32) return false;
  RArgs k{};
  k.row_ptr = a->row_ptr;
  k.col = a->col_idx;
  k.val = a->values;
  k.g = static_cast<const double2*>(s.gsrc);
  k.vin = static_cast<const double2*>(s.vin);
  k.yin = static_cast<const double2*>(s.yin);
  k.out = static_cast<double2*>(s.out);
  k.wout = static_cast<double2*>(s.wout);
  k.ldv = s.ld / epv;
  k.ldyv = s.ld_y / epv;
  k.ldo = s.ld_out / epv;
  k.qv = qv;
  k.row_begin = s.row_begin;
  k.nrows = s.row_end - s.row_begin;
  k.goff = s.goff;
  k.s0 = s.s0;
  k.s1 = s.s1;
  k.s2 = s.s2;
  k.s3 = s.s3;
  k.pol_frac = 1.0f;
  const int pv = ctx->pipe_variant;
  if (cplx) {
    if (a->rp64) dispatch_row<CplxV, int64_t>(ctx, mode, k, pv);
    else dispatch_row<CplxV, int32_t>(ctx, mode, k, pv);
  } else {
    if (a->rp64) dispatch_row<RealV, int64_t>(ctx, mode, k, pv);
    else dispatch_row<RealV, int32_t>(ctx, mode, k, pv);
  }
  return true;
}

}  // namespace adp
