// TMA-pipelined, row-tiled fused Clenshaw step (sm_100a).
//
// Same arithmetic as cheb_step.cu (one degree step of clenshaw_apply,
// proj/src/cheb_filter.cpp:162-177, maspmm + recurrence update fused), but the
// data movement is B200-native:
//   * persistent CTAs walk (panel, row tile) work items in panel-major, row-
//     ascending order, so the front of active rows sweeps the matrix once per
//     panel and the stencil's W reuse stays inside L2;
//   * per tile, ONE elected warp issues TMA bulk copies (cp.async.bulk, SASS
//     UBLKCP) of the tile's metadata blob, of every DISTINCT W row panel the
//     tile touches (the reference's column segments, tiled_matrix.hpp:78-91 --
//     each fetched once per tile instead of once per nonzero) and of the tile's
//     V and Y row panels, all completing on one mbarrier (expect_tx);
//   * a 2-stage shared-memory ring keeps the next tile's copies in flight
//     while the current tile is computed from shared memory, so HBM sees deep
//     memory-level parallelism without register pressure;
//   * the streaming operands (V, Y, outputs) carry an L2 evict-first policy.
// Per row the accumulation is still the CSR (ascending-column) order with
// unfused IEEE ops, so the result is bitwise identical to the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "adp_internal.hpp"

namespace adp {
namespace {

constexpr int kTileWarps = 4;
constexpr int kTileThreads = 32 * kTileWarps;
constexpr int kMaxStages = 8;
constexpr int kMaxDPerLane = 8;  // distinct W rows per tile <= 32 * 8 (tiling cap)

struct TArgs {
  const int32_t* tile_row;
  const int64_t* tile_dptr;
  const int64_t* tile_blob;
  const int32_t* dcol;
  const uint8_t* blob;
  int64_t n_tiles, n_panels, pbv, qv;
  const double2* g;
  const double2* vin;
  const double2* yin;
  double2* out;
  double2* wout;
  int64_t ldv, ldyv, ldo, goff;
  double s0, s1, s2, s3;
  uint32_t stage_bytes;
  int32_t n_stages;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}

__device__ __forceinline__ double2 scale2(double s, double2 a) {
  return make_double2(__dmul_rn(s, a.x), __dmul_rn(s, a.y));
}
__device__ __forceinline__ double2 add2(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 sub2(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}

struct RealT {
  using Val = double;
  static constexpr int kValBytes = 8;
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};
struct CplxT {
  using Val = double2;
  static constexpr int kValBytes = 16;
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

__device__ __forceinline__ uint32_t pad16(uint32_t b) { return (b + 15u) & ~15u; }

struct TileGeom {
  int64_t r0;
  int32_t rows;
  int32_t nd;
  int64_t d0, b0;
  uint32_t bb;
  int32_t pv;  // vectors in this panel
  int64_t panel;
};

__device__ __forceinline__ TileGeom tile_geom(const TArgs& p, int64_t item) {
  TileGeom t;
  t.panel = item / p.n_tiles;
  const int64_t ti = item - t.panel * p.n_tiles;
  t.r0 = __ldg(p.tile_row + ti);
  t.rows = static_cast<int32_t>(__ldg(p.tile_row + ti + 1) - t.r0);
  t.d0 = __ldg(p.tile_dptr + ti);
  t.nd = static_cast<int32_t>(__ldg(p.tile_dptr + ti + 1) - t.d0);
  t.b0 = __ldg(p.tile_blob + ti);
  t.bb = static_cast<uint32_t>(__ldg(p.tile_blob + ti + 1) - t.b0);
  const int64_t rem = p.qv - t.panel * p.pbv;
  t.pv = static_cast<int32_t>(rem < p.pbv ? rem : p.pbv);
  return t;
}

// Per-stage header written by the producer before it arms the stage's
// mbarrier; the consumers read it after the mbarrier wait (acquire).
struct StageHeader {
  int64_t r0, panel;
  int32_t rows, nd, pv;
  uint32_t bb;
};
constexpr uint32_t kHeaderBytes = 32;

// A work item whose geometry and distinct-column list the producer warp has
// prefetched into registers one iteration ahead (hides the dependent loads).
struct Pending {
  int64_t item;
  TileGeom t;
  int32_t cols[kMaxDPerLane];
};

__device__ __forceinline__ void load_pending(const TArgs& p, int64_t item, int64_t total, int lane, Pending& pd) {
  pd.item = item;
  if (item >= total) return;
  pd.t = tile_geom(p, item);
#pragma unroll
  for (int i = 0; i < kMaxDPerLane; ++i) {
    const int idx = lane + 32 * i;
    pd.cols[i] = idx < pd.t.nd ? __ldg(p.dcol + pd.t.d0 + idx) : 0;
  }
}

// Producer: the warp issues every bulk copy of a work item into a stage.
template <bool kStep>
__device__ __forceinline__ void issue_item(const TArgs& p, const Pending& pd, uint8_t* stage, uint64_t* bar,
                                           int lane, uint64_t pol) {
  const TileGeom& t = pd.t;
  const uint32_t pb = static_cast<uint32_t>(t.pv) * 16u;
  const uint32_t total = t.bb + (static_cast<uint32_t>(t.nd) + (kStep ? 2u * t.rows : 0u)) * pb;
  uint8_t* body = stage + kHeaderBytes;
  if (lane == 0) {
    StageHeader* h = reinterpret_cast<StageHeader*>(stage);
    h->r0 = t.r0;
    h->panel = t.panel;
    h->rows = t.rows;
    h->nd = t.nd;
    h->pv = t.pv;
    h->bb = t.bb;
    mbar_arrive_expect_tx(bar, total);
    bulk_g2s(body, p.blob + t.b0, t.bb, bar);
  }
  __syncwarp();
  uint8_t* wst = body + t.bb;
  const int64_t col0 = t.panel * p.pbv;
#pragma unroll
  for (int i = 0; i < kMaxDPerLane; ++i) {
    const int idx = lane + 32 * i;
    if (idx < t.nd)
      bulk_g2s(wst + static_cast<uint32_t>(idx) * pb, p.g + static_cast<int64_t>(pd.cols[i]) * p.ldv + col0, pb,
               bar);
  }
  if constexpr (kStep) {
    uint8_t* vst = wst + static_cast<uint32_t>(t.nd) * pb;
    uint8_t* yst = vst + static_cast<uint32_t>(t.rows) * pb;
    for (int j = lane; j < t.rows; j += 32) {
      bulk_g2s_hint(vst + static_cast<uint32_t>(j) * pb, p.vin + (t.r0 + j) * p.ldv + col0, pb, bar, pol);
      bulk_g2s_hint(yst + static_cast<uint32_t>(j) * pb, p.yin + (t.r0 + j) * p.ldyv + col0, pb, bar, pol);
    }
  }
}

template <class F, int CH, int MODE>
__global__ void __launch_bounds__(kTileThreads, 1) cheb_tile_kernel(const TArgs p) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  using Val = typename F::Val;

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint8_t* stages = smem + 128;
  const int S = p.n_stages;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t total = p.n_tiles * p.n_panels;
  const int64_t grid = gridDim.x;
  const uint64_t pol = policy_evict_first();

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  Pending pend;
  if (warp == 0) {
    for (int s = 0; s < S; ++s) {
      load_pending(p, blockIdx.x + s * grid, total, lane, pend);
      if (pend.item < total) issue_item<kStep>(p, pend, stages + s * p.stage_bytes, &bars[s], lane, pol);
    }
    load_pending(p, blockIdx.x + S * grid, total, lane, pend);  // first re-issue, prefetched
  }

  uint32_t it = 0;
  for (int64_t item = blockIdx.x; item < total; item += grid, ++it) {
    const int s = static_cast<int>(it % S);
    uint8_t* stage = stages + s * p.stage_bytes;
    mbar_wait(&bars[s], (it / S) & 1u);
    const StageHeader h = *reinterpret_cast<const StageHeader*>(stage);
    const uint8_t* body = stage + kHeaderBytes;

    const int32_t* rowoff = reinterpret_cast<const int32_t*>(body);
    const int32_t* own_slot = rowoff + h.rows + 1;
    const int32_t nnz_t = rowoff[h.rows];
    const int32_t* slots = reinterpret_cast<const int32_t*>(body + pad16(4u * (2u * h.rows + 1u)));
    const Val* vals = reinterpret_cast<const Val*>(body + pad16(4u * (2u * h.rows + 1u)) + pad16(4u * nnz_t));
    const double2* wst = reinterpret_cast<const double2*>(body + h.bb);
    const double2* vst = wst + static_cast<int64_t>(h.nd) * h.pv;
    const double2* yst = vst + static_cast<int64_t>(h.rows) * h.pv;
    const int64_t col0 = h.panel * p.pbv;

    bool cv[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) cv[c] = lane + 32 * c < h.pv;

    for (int j = warp; j < h.rows; j += kTileWarps) {
      const int64_t r = h.r0 + j;
      double2 acc[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if constexpr (kSpmmAcc)
          acc[c] = cv[c] ? p.out[r * p.ldo + col0 + lane + 32 * c] : make_double2(0.0, 0.0);
        else
          acc[c] = make_double2(0.0, 0.0);
      }
      const int32_t e1 = rowoff[j + 1];
      for (int32_t e = rowoff[j]; e < e1; ++e) {
        const int32_t sl = slots[e];
        const Val v = vals[e];
        const double2* wrow = wst + static_cast<int64_t>(sl) * h.pv;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          if (!cv[c]) continue;
          double2 w = wrow[lane + 32 * c];
          if constexpr (kFirst) w = scale2(p.s2, w);
          acc[c] = F::mac(acc[c], v, w);
        }
      }
      double2 own[CH];
      if constexpr (kNeedOwn) {
        const int32_t os = own_slot[j];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          if (!cv[c]) continue;
          double2 w = os >= 0 ? wst[static_cast<int64_t>(os) * h.pv + lane + 32 * c]
                              : __ldg(p.g + (r + p.goff) * p.ldv + col0 + lane + 32 * c);
          if constexpr (kFirst) w = scale2(p.s2, w);
          own[c] = w;
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (!cv[c]) continue;
        double2 res;
        if constexpr (kStep) {
          const double2 vv = vst[static_cast<int64_t>(j) * h.pv + lane + 32 * c];
          const double2 yy = yst[static_cast<int64_t>(j) * h.pv + lane + 32 * c];
          res = add2(sub2(add2(scale2(p.s0, acc[c]), scale2(p.s1, own[c])), vv), scale2(p.s2, yy));
        } else if constexpr (kFirst) {
          st_hint(p.wout + r * p.ldo + col0 + lane + 32 * c, own[c], pol);
          res = add2(scale2(p.s0, acc[c]), scale2(p.s1, own[c]));
        } else if constexpr (kDeg1) {
          res = add2(scale2(p.s0, own[c]), scale2(p.s1, add2(scale2(p.s2, acc[c]), scale2(p.s3, own[c]))));
        } else {
          res = acc[c];
        }
        st_hint(p.out + r * p.ldo + col0 + lane + 32 * c, res, pol);
      }
    }
    __syncthreads();  // every warp is done with this stage
    if (warp == 0 && pend.item < total) {
      issue_item<kStep>(p, pend, stage, &bars[s], lane, pol);
      load_pending(p, pend.item + grid, total, lane, pend);
    }
  }
}

template <class F, int CH>
void launch_tile(adp_ctx* ctx, StepMode mode, const TArgs& k, size_t smem, int ctas_per_sm) {
  static size_t configured[5] = {0, 0, 0, 0, 0};
  auto run = [&](auto kern, int m) {
    if (configured[m] < smem) {
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      configured[m] = smem;
    }
    const int64_t items = k.n_tiles * k.n_panels;
    const int grid = static_cast<int>(std::min<int64_t>(items, static_cast<int64_t>(ctx->sm_count) * ctas_per_sm));
    kern<<<grid, kTileThreads, smem, ctx->stream>>>(k);
  };
  switch (mode) {
    case StepMode::First: run(cheb_tile_kernel<F, CH, 0>, 0); break;
    case StepMode::Step: run(cheb_tile_kernel<F, CH, 1>, 1); break;
    case StepMode::Deg1: run(cheb_tile_kernel<F, CH, 2>, 2); break;
    case StepMode::Spmm: run(cheb_tile_kernel<F, CH, 3>, 3); break;
    case StepMode::SpmmAcc: run(cheb_tile_kernel<F, CH, 4>, 4); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

}  // namespace

bool launch_step_tiled(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  adp_csr* a = const_cast<adp_csr*>(s.a);
  const bool cplx = a->dtype == ADP_C128;
  const int epv = cplx ? 1 : 2;
  const int64_t qv = (s.q + epv - 1) / epv;
  if (qv < 32) return false;  // thin blocks: the row kernel's narrow groups fit better
  if (s.row_begin != 0 || s.row_end != a->n_rows) return false;  // partial row ranges use the row kernel
  // panel width: up to ch_cap vectors per lane, balanced over panels
  const int64_t ch_cap = ctx->tile_ch > 0 ? ctx->tile_ch : 4;
  const int64_t n_panels = (qv + 32 * ch_cap - 1) / (32 * ch_cap);
  const int64_t ch = ((qv + n_panels - 1) / n_panels + 31) / 32;
  const int64_t pbv = 32 * ch;
  const int stages = std::max(2, std::min(kMaxStages, ctx->tile_stages > 0 ? ctx->tile_stages : 4));
  const int64_t stage_bytes = static_cast<int64_t>(ctx->tile_stage_kb > 0 ? ctx->tile_stage_kb : 54) * 1024;
  const int ctas = ctx->tile_ctas > 0 ? ctx->tile_ctas : 1;
  if (128 + stages * stage_bytes > 227 * 1024 / ctas) return false;
  const Tiling* t = get_tiling(a, pbv * 16, stage_bytes - kHeaderBytes);
  if (!t) return false;
  TArgs k{};
  k.tile_row = static_cast<const int32_t*>(t->d_tile_row);
  k.tile_dptr = static_cast<const int64_t*>(t->d_tile_dptr);
  k.tile_blob = static_cast<const int64_t*>(t->d_tile_blob);
  k.dcol = static_cast<const int32_t*>(t->d_dcol);
  k.blob = static_cast<const uint8_t*>(t->d_blob);
  k.n_tiles = t->n_tiles;
  k.n_panels = (qv + pbv - 1) / pbv;
  k.pbv = pbv;
  k.qv = qv;
  k.g = static_cast<const double2*>(s.gsrc);
  k.vin = static_cast<const double2*>(s.vin);
  k.yin = static_cast<const double2*>(s.yin);
  k.out = static_cast<double2*>(s.out);
  k.wout = static_cast<double2*>(s.wout);
  k.ldv = s.ld / epv;
  k.ldyv = s.ld_y / epv;
  k.ldo = s.ld_out / epv;
  k.goff = s.goff;
  k.s0 = s.s0;
  k.s1 = s.s1;
  k.s2 = s.s2;
  k.s3 = s.s3;
  k.stage_bytes = static_cast<uint32_t>(stage_bytes);
  k.n_stages = stages;
  const size_t smem = 128 + static_cast<size_t>(stages) * stage_bytes;
  if (cplx) {
    switch (ch) {
      case 1: launch_tile<CplxT, 1>(ctx, mode, k, smem, ctas); break;
      case 2: launch_tile<CplxT, 2>(ctx, mode, k, smem, ctas); break;
      case 3: launch_tile<CplxT, 3>(ctx, mode, k, smem, ctas); break;
      default: launch_tile<CplxT, 4>(ctx, mode, k, smem, ctas); break;
    }
  } else {
    switch (ch) {
      case 1: launch_tile<RealT, 1>(ctx, mode, k, smem, ctas); break;
      case 2: launch_tile<RealT, 2>(ctx, mode, k, smem, ctas); break;
      case 3: launch_tile<RealT, 3>(ctx, mode, k, smem, ctas); break;
      default: launch_tile<RealT, 4>(ctx, mode, k, smem, ctas); break;
    }
  }
  return true;
}

}  // namespace adp
