// Two Clenshaw degree steps in one launch ("pair" kernel), sm_100a.
//
// clenshaw_apply (proj/src/cheb_filter.cpp:166-177) runs, per degree step j,
//     b_j = ((s0 * A b_{j+1} + s1 * b_{j+1}) - b_{j+2}) + c_j * y
// and every step streams four n x q blocks through HBM (gathered b_{j+1}, b_{j+2},
// y, the written b_j). Step j-1 needs b_j only at the rows its CSR rows touch, so
// a sweep of step j-1 that trails the sweep of step j by more than the operator's
// row reach can consume b_j -- and the b_{j+1} / y rows step j just read -- while
// they are still in the 126 MB L2. Per pair of steps HBM then sees b_{j+1} and
// b_{j+2} and y read once and b_j and b_{j-1} written once: 5 block streams
// instead of 8. Every element is computed by the same expression in the same
// order as the single-step kernel: results are bitwise identical.
//
// Schedule: rows are cut into chunks of WARPS rows (one row per warp, the lean
// kernel's mapping). Per column panel the tickets are
//     F_0 .. F_{D-1}, then F_{D}, B_0, F_{D+1}, B_1, ..., then the remaining B
// (F = chunk of step j, B = chunk of step j-1), assigned round-robin to a
// persistent, co-resident grid (cooperative launch). B_k waits until every F
// chunk in the groups of chunks its rows read (RAW on b_j) or whose rows read the
// b_{j+1} rows it overwrites (WAR, in-place output) has published completion on
// a per-group counter. D exceeds the largest such reach, so every awaited F
// ticket is smaller than B_k's: the smallest unfinished ticket can always run
// (no deadlock), and with D's slack of about half the grid the waits are rare.
//
// Coherence: b_j is written inside the launch, so the step-(j-1) gathers and own
// row read it with ld.global.cg (L2), never through the non-coherent/L1 path.
// Completion: __syncthreads, then one thread adds to the counter with release
// semantics (cumulative over the CTA's stores, the cooperative-groups grid-sync
// pattern); waiters poll with relaxed loads, then __syncthreads.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

PairPlan::~PairPlan() {
  cudaFree(d_glo);
  cudaFree(d_ghi);
  cudaFree(d_counters);
}

namespace {

struct PArgs {
  const void* row_ptr;
  const int32_t* col;
  const void* val;
  const char* A;  // b_{j+1}: step-j gathers and own row; step-(j-1) V operand
  char* B;        // b_{j+2} in, b_j out (step j, in place)
  const char* y;
  char* out;      // b_{j-1} (== A for the in-place middle steps)
  uint32_t ld_b, ldy_b, ldo_b;
  int32_t nrows, nch, n_panels, D, grid;
  int32_t gs;                // chunks per counter group
  int32_t ngroups;
  const int32_t* glo;        // per chunk: first / last counter group a B chunk waits on
  const int32_t* ghi;
  uint32_t* counters;        // [n_panels][ngroups], cumulative over launches
  uint32_t epoch;            // this launch's number (>= 1)
  double f0, f1, f2;         // step j scalars
  double b0, b1, b2;         // step j-1 scalars
};

struct RealP {
  using Val = double;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double*>(p) + k); }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};
struct CplxP {
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
  uint64_t pol;
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void st_hint(void* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_plain(void* p, double2 v) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// Counter loads are relaxed (no L1 invalidation per poll, which an acquire load
// costs): every load of data produced inside the launch is an L2 (.cg) load
// issued after the poll returned, and the producer publishes with a release.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
template <class RP>
__device__ __forceinline__ int64_t ld_rp(const void* p, int64_t i) {
  return static_cast<int64_t>(__ldg(static_cast<const RP*>(p) + i));
}

// Ticket t of a panel -> (is step j-1, chunk).
__device__ __forceinline__ void decode(int32_t t, int32_t nch, int32_t D, bool& back, int32_t& k) {
  if (t < D) {
    back = false;
    k = t;
    return;
  }
  const int32_t u = t - D, m = nch - D;
  if (u < 2 * m) {
    back = u & 1;
    k = back ? (u >> 1) : D + (u >> 1);
  } else {
    back = true;
    k = m + (u - 2 * m);
  }
}

template <class F, int CH, int WARPS, class RP, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) cheb_pair_kernel(const PArgs p) {
  constexpr uint32_t kPB = 32 * CH * 16u;
  using Val = typename F::Val;
  extern __shared__ __align__(16) uint8_t smem[];  // [WARPS mbarriers | pad][warp][V, Y]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp;
  double2* my = reinterpret_cast<double2*>(smem + 128) + warp * (2 * 32 * CH);
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  const uint64_t pol = policy_evict_first(1.0f);
  const int32_t per_panel = 2 * p.nch;
  const int32_t total = per_panel * p.n_panels;
  for (int32_t T = blockIdx.x; T < total; T += p.grid) {
    const int32_t panel = T / per_panel;
    bool back;
    int32_t k;
    decode(T - panel * per_panel, p.nch, p.D, back, k);
    const int32_t r32 = k * WARPS + warp;
    const bool live = r32 < p.nrows;
    const int64_t r = r32;
    const uint32_t poff = static_cast<uint32_t>(panel) * kPB;
    const uint32_t voff = poff + lane * 16u;
    const char* gsrc = back ? p.B : p.A;   // gathered operand
    const char* vsrc = back ? p.A : p.B;   // previous-previous iterate
    if (live && lane == 0) {
      mbar_arrive_expect_tx(bar, 2 * kPB);
      bulk_g2s_hint(my, vsrc + static_cast<uint64_t>(r) * p.ld_b + poff, kPB, bar, pol);
      if (back)
        bulk_g2s_hint(my + 32 * CH, p.y + static_cast<uint64_t>(r) * p.ldy_b + poff, kPB, bar, pol);
      else
        bulk_g2s(my + 32 * CH, p.y + static_cast<uint64_t>(r) * p.ldy_b + poff, kPB, bar);  // kept for step j-1
    }
    if (back) {  // CTA-uniform: wait for the step-j chunks this chunk depends on
      const int32_t g0 = __ldg(p.glo + k), g1 = __ldg(p.ghi + k);
      uint32_t* cnt = p.counters + static_cast<int64_t>(panel) * p.ngroups;
      for (int32_t g = g0 + static_cast<int32_t>(threadIdx.x); g <= g1; g += WARPS * 32) {
        const int32_t size = min(p.gs, p.nch - g * p.gs);
        const uint32_t target = p.epoch * static_cast<uint32_t>(size);
        while (static_cast<int32_t>(ld_relaxed(cnt + g) - target) < 0) __nanosleep(64);
      }
      __syncthreads();
    }
    if (live) {
      double2 acc[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = make_double2(0.0, 0.0);
      const char* gb = gsrc + voff;
      const RP start = static_cast<RP>(ld_rp<RP>(p.row_ptr, r));
      const RP end = static_cast<RP>(ld_rp<RP>(p.row_ptr, r + 1));
      for (RP e = start; e < end; ++e) {
        const int cidx = __ldg(p.col + e);
        const Val v = F::load(p.val, static_cast<int64_t>(e));
        const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cidx)) * p.ld_b);
        double2 w[CH];
        if (back) {
#pragma unroll
          for (int c = 0; c < CH; ++c) w[c] = __ldcg(src + 32 * c);
        } else {
#pragma unroll
          for (int c = 0; c < CH; ++c) w[c] = __ldg(src + 32 * c);
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = F::mac(acc[c], v, w[c]);
      }
      __syncwarp();
      mbar_wait(bar, phase);
      phase ^= 1u;
      const double2* own_src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(r) * p.ld_b);
      const double s0 = back ? p.b0 : p.f0, s1 = back ? p.b1 : p.f1, s2 = back ? p.b2 : p.f2;
      char* ob = back ? p.out + static_cast<uint64_t>(r) * p.ldo_b + voff : p.B + static_cast<uint64_t>(r) * p.ld_b + voff;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const double2 own = back ? __ldcg(own_src + 32 * c) : __ldg(own_src + 32 * c);
        const double2 vv = my[c * 32 + lane];
        const double2 yy = my[32 * CH + c * 32 + lane];
        // v = (((s0 * aw) + (s1 * w)) - v) + (s2 * y)   (cheb_filter.cpp:170-171, 176-177)
        const double2 res = add2(sub2(add2(scale2(s0, acc[c]), scale2(s1, own)), vv), scale2(s2, yy));
        if (back)
          st_hint(ob + 512 * c, res, pol);
        else
          st_plain(ob + 512 * c, res);  // b_j: gathered by step j-1 from L2
      }
      __syncwarp();  // the slot is refilled by the next ticket's copy
    }
    if (!back) {  // publish the chunk
      __syncthreads();
      if (threadIdx.x == 0) red_release_add(p.counters + static_cast<int64_t>(panel) * p.ngroups + k / p.gs, 1u);
    }
  }
}

template <class F, int CH, int WARPS, class RP, int MINB>
bool launch_pair_cfg(adp_ctx* ctx, const adp_csr* a, const PairStep& ps, int64_t qv, int slack_pct) {
  constexpr int64_t kGS = 64;
  if (qv % (32 * CH) != 0) return false;
  const int64_t n = a->n_rows;
  const int64_t nch = (n + WARPS - 1) / WARPS;
  const int64_t n_panels = qv / (32 * CH);
  if (2 * nch * n_panels >= (int64_t{1} << 31) || n >= (int64_t{1} << 31)) return false;
  PairPlan* plan = get_pair_plan(const_cast<adp_csr*>(a), WARPS, kGS, n_panels);
  auto kern = cheb_pair_kernel<F, CH, WARPS, RP, MINB>;
  const size_t smem = 128 + static_cast<size_t>(WARPS) * 2 * 32 * CH * 16;
  if (smem > 48 * 1024)
    ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  ADP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem));
  if (per_sm < 1) return false;
  const int64_t tickets = 2 * nch * n_panels;
  const int grid = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(per_sm) * ctx->sm_count, tickets));
  // lag: the largest reach (in chunks, rounded to whole groups) plus slack for
  // the tickets in flight (about half the grid are step-j chunks)
  const int64_t slack = static_cast<int64_t>(grid) * slack_pct / 100;
  const int64_t D = std::min<int64_t>(nch, plan->reach + kGS + 1 + slack);
  PArgs p{};
  p.row_ptr = a->row_ptr;
  p.col = a->col_idx;
  p.val = a->values;
  const int64_t eb = a->dtype == ADP_C128 ? 16 : 8;
  p.A = static_cast<const char*>(ps.g);
  p.B = static_cast<char*>(ps.v);
  p.y = static_cast<const char*>(ps.y);
  p.out = static_cast<char*>(ps.out);
  p.ld_b = static_cast<uint32_t>(ps.ld * eb);
  p.ldy_b = static_cast<uint32_t>(ps.ld_y * eb);
  p.ldo_b = static_cast<uint32_t>(ps.ld_out * eb);
  p.nrows = static_cast<int32_t>(n);
  p.nch = static_cast<int32_t>(nch);
  p.n_panels = static_cast<int32_t>(n_panels);
  p.D = static_cast<int32_t>(D);
  p.grid = grid;
  p.gs = static_cast<int32_t>(kGS);
  p.ngroups = static_cast<int32_t>(plan->ngroups);
  p.glo = static_cast<const int32_t*>(plan->d_glo);
  p.ghi = static_cast<const int32_t*>(plan->d_ghi);
  p.counters = static_cast<uint32_t*>(plan->d_counters);
  p.epoch = ++plan->epoch;
  p.f0 = ps.f0;
  p.f1 = ps.f1;
  p.f2 = ps.f2;
  p.b0 = ps.b0;
  p.b1 = ps.b1;
  p.b2 = ps.b2;
  void* args[] = {&p};
  ADP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(WARPS * 32), args, smem,
                                       ctx->stream));
  ctx->launches += 1;
  return true;
}

template <class F, class RP>
bool dispatch_pair(adp_ctx* ctx, const adp_csr* a, const PairStep& ps, int64_t qv) {
  switch (ctx->pair_variant) {
    case 1: return launch_pair_cfg<F, 4, 8, RP, 4>(ctx, a, ps, qv, 50);
    case 2: return launch_pair_cfg<F, 2, 8, RP, 4>(ctx, a, ps, qv, 50);
    case 3: return launch_pair_cfg<F, 1, 8, RP, 6>(ctx, a, ps, qv, 50);
    case 4: return launch_pair_cfg<F, 2, 8, RP, 4>(ctx, a, ps, qv, 25);
    case 5: return launch_pair_cfg<F, 1, 8, RP, 6>(ctx, a, ps, qv, 25);
    case 6: return launch_pair_cfg<F, 1, 8, RP, 6>(ctx, a, ps, qv, 100);
    default: return false;
  }
}

}  // namespace

// Chunk dependency plan of an operator for the pair kernel: for chunk k (rows
// [k*C, (k+1)*C)) the range of step-j chunks that must be complete before step
// j-1 may run on it -- the chunks holding the columns its rows read, and the
// chunks whose rows read its rows' (overwritten) b_{j+1} values -- as counter
// groups, plus the largest forward reach.
PairPlan* get_pair_plan(adp_csr* a, int64_t chunk_rows, int64_t gs, int64_t n_panels) {
  PairPlan* plan = nullptr;
  for (auto& p : a->pair_plans)
    if (p->chunk_rows == chunk_rows && p->gs == gs) plan = p.get();
  if (!plan) {
    auto p = std::make_unique<PairPlan>();
    p->chunk_rows = chunk_rows;
    p->gs = gs;
    const int64_t n = a->n_rows;
    const int64_t nch = (n + chunk_rows - 1) / chunk_rows;
    std::vector<int64_t> lo(nch), hi(nch);
    for (int64_t k = 0; k < nch; ++k) lo[k] = hi[k] = k;
    ensure_host_copy(const_cast<adp_csr*>(a));
    const std::vector<int64_t>& rp = a->h_row_ptr;
    const std::vector<int32_t>& ci = a->h_col;
    for (int64_t r = 0; r < n; ++r) {
      const int64_t kr = r / chunk_rows;
      for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
        const int64_t kc = ci[e] / chunk_rows;
        lo[kr] = std::min(lo[kr], kc);  // RAW: rows of kr read b_j rows in chunk kc
        hi[kr] = std::max(hi[kr], kc);
        lo[kc] = std::min(lo[kc], kr);  // WAR: rows of kr read b_{j+1} rows of kc
        hi[kc] = std::max(hi[kc], kr);
      }
    }
    const int64_t ngroups = (nch + gs - 1) / gs;
    std::vector<int32_t> glo(nch), ghi(nch);
    int64_t reach = 0;
    for (int64_t k = 0; k < nch; ++k) {
      glo[k] = static_cast<int32_t>(lo[k] / gs);
      ghi[k] = static_cast<int32_t>(hi[k] / gs);
      reach = std::max(reach, hi[k] - k);
    }
    p->nch = nch;
    p->ngroups = ngroups;
    p->reach = reach;
    ADP_CUDA(cudaSetDevice(a->ctx->device));
    ADP_CUDA(cudaMalloc(&p->d_glo, std::max<size_t>(nch * 4, 16)));
    ADP_CUDA(cudaMalloc(&p->d_ghi, std::max<size_t>(nch * 4, 16)));
    ADP_CUDA(cudaMemcpy(p->d_glo, glo.data(), nch * 4, cudaMemcpyHostToDevice));
    ADP_CUDA(cudaMemcpy(p->d_ghi, ghi.data(), nch * 4, cudaMemcpyHostToDevice));
    plan_uploads_done();
    a->pair_plans.push_back(std::move(p));
    plan = a->pair_plans.back().get();
  }
  if (plan->counter_panels < n_panels) {  // (re)allocate zeroed counters; epochs restart
    ADP_CUDA(cudaStreamSynchronize(a->ctx->stream));
    cudaFree(plan->d_counters);
    plan->d_counters = nullptr;
    const size_t bytes = static_cast<size_t>(n_panels * plan->ngroups) * 4;
    ADP_CUDA(cudaMalloc(&plan->d_counters, std::max<size_t>(bytes, 16)));
    ADP_CUDA(cudaMemset(plan->d_counters, 0, std::max<size_t>(bytes, 16)));
    plan->counter_panels = n_panels;
    plan->epoch = 0;
  }
  return plan;
}

bool launch_pair(adp_ctx* ctx, const adp_csr* a, const PairStep& ps, int64_t q) {
  if (ctx->pair_variant == 0 || a->n_rows != a->n_cols) return false;
  const bool cplx = a->dtype == ADP_C128;
  const int64_t eb = cplx ? 16 : 8;
  const int epv = cplx ? 1 : 2;
  if (q % epv != 0) return false;
  const int64_t qv = q / epv;
  for (int64_t ld : {ps.ld, ps.ld_y, ps.ld_out})
    if ((ld * eb) % 16 != 0 || ld * eb >= (int64_t{1} << 32)) return false;
  for (const void* ptr : {ps.g, static_cast<const void*>(ps.v), ps.y, static_cast<const void*>(ps.out)})
    if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0) return false;
  if (cplx) return a->rp64 ? dispatch_pair<CplxP, int64_t>(ctx, a, ps, qv) : dispatch_pair<CplxP, int32_t>(ctx, a, ps, qv);
  return a->rp64 ? dispatch_pair<RealP, int64_t>(ctx, a, ps, qv) : dispatch_pair<RealP, int32_t>(ctx, a, ps, qv);
}

}  // namespace adp
