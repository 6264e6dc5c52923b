// Fused Clenshaw step for banded operators with sparse off-band entries (config 5): the band-block
// ("band") kernel, sm_100a.
//
// Config 5's rows hold a dense band [r - h, r + h] (h = 250: 501 entries) plus ~40 random entries
// outside it. The lean kernel gathers every entry's W row panel through L1 per output row: 541 row
// panels per row, 13.3 TB of L1 traffic per degree step (L1-throughput bound, 606 ms). Consecutive
// rows' bands overlap in all but one column, so here a warp owns R consecutive rows of one column
// panel and sweeps the UNION of their bands once, column by column: each W row panel is loaded once
// (into registers) and applied to all R rows whose band holds that column -- R times less gather
// traffic, and R independent accumulator sets per lane for the FP64 pipe.
//
// Per row the products still accumulate in ascending column order -- its lower off-band entries
// (before the sweep), its band (during the sweep, column ascending), its upper off-band entries
// (after it) -- which is CSR order, so the result is bitwise the lean kernel's (complex: four
// DFMA per entry, the order the complex path defines; real: the reference's unfused mul + add).
//
// What makes it run (each step measured on config 5 at full size): the band's operator
// values are loaded coalesced one chunk AHEAD and read back from the warp's shared-memory slot as
// broadcasts with compile-time offsets (values loaded at use: 1051 ms; staged: 485-522 ms); the
// off-band W row panels -- random rows, each a DRAM round trip -- land through a ring of cp.async stages
// in the same slot, L1 bypassed; and ONE gather code path serves both off-band phases, because at 52K
// instructions the kernel fell out of the instruction cache (743 ms; compact: 391-417 ms, power-bound).
//
// The host derives h from the middle row and a device kernel verifies, for EVERY row, that its
// columns are [lower off-band | max(0, r - h) .. min(n - 1, r + h) | upper off-band] and records
// the number of lower entries (BandPlan, once per operator: config 5's 43 GB operator is generated
// on the device and is never copied to the host for this).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

BandPlan::~BandPlan() { cudaFree(d_nlow); }

namespace {

template <class RP>
__global__ void band_plan_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col, int64_t n, int64_t h,
                                 int32_t* __restrict__ nlow, int* __restrict__ bad) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e0 = rp[r], e1 = rp[r + 1];
    const int64_t b0 = r - h < 0 ? 0 : r - h, b1 = r + h > n - 1 ? n - 1 : r + h, len = b1 - b0 + 1;
    int64_t lo = e0, hi = e1;  // first entry with column >= b0
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (col[mid] < b0) lo = mid + 1;
      else hi = mid;
    }
    // columns are strictly ascending (checked at upload): b0 at lo and b1 at lo + len - 1 means the
    // whole band is present
    const bool ok = lo + len <= e1 && col[lo] == b0 && col[lo + len - 1] == b1 && lo - e0 < (int64_t{1} << 31);
    if (!ok) atomicExch(bad, 1);
    nlow[r] = static_cast<int32_t>(lo - e0);
  }
}

struct RealB {
  using Val = double;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double*>(p) + k); }
  static __device__ __forceinline__ Val ldp(const Val* p) { return __ldg(p); }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};
struct CplxB {
  using Val = double2;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double2*>(p) + k); }
  static __device__ __forceinline__ Val ldp(const Val* p) { return __ldg(p); }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {  // as CplxL::mac (cheb_lean.cu)
    acc.x = __fma_rn(v.x, w.x, acc.x);
    acc.x = __fma_rn(-v.y, w.y, acc.x);
    acc.y = __fma_rn(v.x, w.y, acc.y);
    acc.y = __fma_rn(v.y, w.x, acc.y);
    return acc;
  }
};

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_hint(void* ptr, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ double2 ld_nc(const char* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
template <class RP>
__device__ __forceinline__ int64_t ld_rp(const void* p, int64_t i) {
  return static_cast<int64_t>(__ldg(static_cast<const RP*>(p) + i));
}

struct BArgs {
  const void* row_ptr;
  const int32_t* col;
  const void* val;
  const int32_t* nlow;
  const char* g;  // W (gathered)
  const char* vin;
  const char* yin;
  char* out;
  uint32_t ldg_b, ldy_b, ldo_b;  // row pitches in bytes
  int64_t n;
  int32_t h, n_blocks, n_panels, valid;  // valid: 16-byte vectors per row that exist
  double s0, s1, s2;
};

constexpr int kCH = 2;  // 16-byte vectors per lane: a panel is 32 x kCH vectors (1 KB per row)
constexpr int kPF = 2;  // band sweep: W row panels loaded this many columns ahead

__device__ __forceinline__ double shfl_val(double v, int j) { return __shfl_sync(0xffffffffu, v, j); }
__device__ __forceinline__ double2 shfl_val(double2 v, int j) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, j), __shfl_sync(0xffffffffu, v.y, j));
}
__device__ __forceinline__ double zero_val(double) { return 0.0; }
__device__ __forceinline__ double2 zero_val(double2) { return make_double2(0.0, 0.0); }

// Off-band entries [e0, e0 + cnt) of GR consecutive rows (warp-uniform e0 / cnt per row), entry by
// entry in CSR order per row, the GR rows interleaved so GR x kCH gathers are in flight. Columns and
// values are fetched 32 entries at a time (coalesced) and handed out by shuffles.

// 16-byte asynchronous copy global -> shared, bypassing L1 (the gathered rows are used once);
// bytes = 0 writes zeros without reading.
__device__ __forceinline__ void cp_async16(uint32_t dst, const char* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ double2 lds128(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}

// Off-band entries [e0, e0 + cnt) of GR consecutive rows (warp-uniform e0 / cnt per row), entry by
// entry in CSR order per row, the GR rows interleaved. Columns and values are fetched 32 entries at a
// time (coalesced) and handed out by shuffles. The gathered W row panels are random rows of a block
// far larger than L2 -- each a DRAM round trip -- so they land through a ring of D stages of
// asynchronous copies in the warp's shared-memory slot (each lane copies and reads back its own 16
// bytes: no cross-lane ordering): D x GR row panels are in flight per warp without holding registers,
// and the gathers bypass L1, which keeps the band's W rows.
template <class F, int GR, int D>
__device__ __forceinline__ void offband(const BArgs& p, const char* gb, uint32_t ring,
                                        const bool (&ok)[kCH], const int64_t (&e0)[GR], const int32_t (&cnt)[GR],
                                        double2 (*acc)[kCH], int lane) {
  using Val = typename F::Val;
  int32_t maxcnt = 0;
#pragma unroll
  for (int g = 0; g < GR; ++g) maxcnt = cnt[g] > maxcnt ? cnt[g] : maxcnt;
  constexpr uint32_t kStage = GR * kCH * 512;        // bytes of one ring stage
  for (int32_t base = 0; base < maxcnt; base += 32) {
    int32_t mc[GR];
    Val mv[GR];
#pragma unroll
    for (int g = 0; g < GR; ++g) {
      const bool in = base + lane < cnt[g];
      mc[g] = in ? __ldg(p.col + e0[g] + base + lane) : 0;
      mv[g] = in ? F::load(p.val, e0[g] + base + lane) : zero_val(Val{});
    }
    const int32_t lim = maxcnt - base < 32 ? maxcnt - base : 32;
    auto issue = [&](int32_t j) {  // entry j of every row -> stage j % D (zeros where a row has no j-th entry)
      const uint32_t dst = ring + static_cast<uint32_t>(j % D) * kStage + lane * 16;
#pragma unroll
      for (int g = 0; g < GR; ++g) {
        const bool in = j < 32 && base + j < cnt[g];  // warp-uniform
        const char* src = gb + static_cast<uint64_t>(static_cast<uint32_t>(__shfl_sync(0xffffffffu, mc[g], j & 31))) * p.ldg_b;
#pragma unroll
        for (int c = 0; c < kCH; ++c) cp_async16(dst + (g * kCH + c) * 512, src + c * 512, in && ok[c] ? 16u : 0u);
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int t = 0; t < D - 1; ++t) issue(t);
#pragma unroll 1
    for (int32_t j = 0; j < lim; ++j) {
      issue(j + D - 1);  // stage (j - 1) % D: its reads finished with iteration j - 1's MACs
      cp_async_wait<D - 1>();
      // A row without a j-th entry takes v = 0 (the zero fill above) and w = 0 (zero-filled copy):
      // acc + 0 * 0 == acc bit for bit (acc is never -0)
      const uint32_t st = ring + static_cast<uint32_t>(j % D) * kStage + lane * 16;
      double2 w[GR][kCH];
      Val v[GR];
#pragma unroll
      for (int g = 0; g < GR; ++g) {
        v[g] = shfl_val(mv[g], j);
#pragma unroll
        for (int c = 0; c < kCH; ++c) w[g][c] = lds128(st + (g * kCH + c) * 512);
      }
#pragma unroll
      for (int g = 0; g < GR; ++g)
#pragma unroll
        for (int c = 0; c < kCH; ++c) acc[g][c] = F::mac(acc[g][c], v[g], w[g][c]);
    }
    cp_async_wait<0>();
  }
}

template <class F, int R, int KC, int GR, int D>
struct BandSlot {
  static constexpr uint32_t ring = D * GR * kCH * 512, vals = R * KC * sizeof(typename F::Val);
  static constexpr uint32_t bytes = ring > vals ? ring : vals;
};

// One warp per (block of R consecutive rows, panel of 32 x kCH 16-byte vectors); Step mode. A CTA's
// warps take consecutive row blocks of ONE panel (they sweep nearly the same W rows: L1 hits), and
// consecutive CTAs take the panels of one row group (they stream the same operator values: L2 hits).
//
// Band sweep: the union of the R bands in chunks of KC columns. A chunk's R x KC operator values are
// loaded coalesced one chunk AHEAD (registers), parked in the warp's shared-memory slot and read back
// as broadcasts with compile-time offsets, so the inner loop is: one W row panel (loaded kPF columns
// ahead), R broadcast value reads, R x kCH MACs. Chunks inside every row's band (all but the first
// and last one or two) run without per-entry checks.
template <class F, int R, int KC, class RP, int NT, int MINB, int GR, int D>
__global__ void __launch_bounds__(NT, MINB) cheb_band_kernel(const BArgs p) {
  using Val = typename F::Val;
  static_assert(R % GR == 0 && D >= 2, "band kernel gather geometry");
  constexpr int NW = NT / 32;
  constexpr int NV = R * KC / 32;  // values per lane and chunk
  constexpr int RPJ = 32 / KC;     // rows covered by one 32-lane load
  static_assert(KC <= 32 && 32 % KC == 0 && (R * KC) % 32 == 0 && KC % kPF == 0, "band kernel geometry");
  // per warp: the gather ring (off-band phases), reused as the value chunk slot (band sweep)
  constexpr uint32_t kSlot = BandSlot<F, R, KC, GR, D>::bytes;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Val* sm = reinterpret_cast<Val*>(smem_raw + warp * kSlot);
  const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const int64_t group = blockIdx.x / p.n_panels;
  const int panel = static_cast<int>(blockIdx.x - group * p.n_panels);
  const int64_t r0 = (group * NW + warp) * R;
  if (r0 >= p.n) return;  // warp-uniform; no CTA-wide barrier below
  const uint32_t voff = (static_cast<uint32_t>(panel) * 32 * kCH + lane) * 16u;
  bool ok[kCH];
#pragma unroll
  for (int c = 0; c < kCH; ++c) ok[c] = panel * 32 * kCH + c * 32 + lane < p.valid;
  const bool full_panel = (panel + 1) * 32 * kCH <= p.valid;
  const int32_t h = p.h;
  const int32_t n32 = static_cast<int32_t>(p.n);
  const int32_t rr0 = static_cast<int32_t>(r0);
  const int32_t rows = n32 - rr0 < R ? n32 - rr0 : R;  // rows of this block that exist
  // union of the bands: [cs, ce)
  const int32_t cs = rr0 - h < 0 ? 0 : rr0 - h;
  const int32_t ce = (rr0 + rows - 1 + h > n32 - 1 ? n32 - 1 : rr0 + rows - 1 + h) + 1;
  const int32_t n_chunks = (ce - cs + KC - 1) / KC;
  // chunks [m_lo, m_hi) lie inside every row's band and need no checks (full blocks and panels only)
  int32_t m_lo = 0, m_hi = 0;
  if (rows == R && full_panel) {
    const int32_t ilo = rr0 + R - 1 - h < 0 ? 0 : rr0 + R - 1 - h;             // last row's first column
    const int32_t ihi = (rr0 + h > n32 - 1 ? n32 - 1 : rr0 + h) + 1;           // first row's end
    const int32_t lim = ihi < n32 - kPF ? ihi : n32 - kPF;                     // the W prefetch stays inside W
    m_lo = (ilo - cs + KC - 1) / KC;
    m_hi = lim - cs >= 0 ? (lim - cs) / KC : 0;
    if (m_hi < m_lo) m_hi = m_lo;
  }
  // this lane's rows of a chunk load: value j is row (j RPJ + lane / KC), column k = lane % KC;
  // vp[j] + cc addresses the entry of column cc
  const int kl = lane % KC;
  const Val* vp[NV];
  int32_t vlo[NV], vhi[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int32_t r = rr0 + j * RPJ + lane / KC;
    const int32_t rc = r < n32 ? r : n32 - 1;
    const int32_t lo = rc - h < 0 ? 0 : rc - h;
    vlo[j] = lo;
    vhi[j] = r < n32 ? (rc + h > n32 - 1 ? n32 - 1 : rc + h) + 1 : lo;  // empty for rows past the end
    vp[j] = static_cast<const Val*>(p.val) + (ld_rp<RP>(p.row_ptr, rc) + __ldg(p.nlow + rc) - lo);
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const char* gb = p.g + voff;
  double2 acc[R][kCH];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int c = 0; c < kCH; ++c) acc[i][c] = make_double2(0.0, 0.0);

  // Phases: 0 = lower off-band entries (they precede the band in every row's column order) and the
  // band sweep, 1 = upper off-band entries. One loop so the gather code exists once (the kernel must
  // stay inside the instruction cache: three warps per scheduler sit at different phases).
#pragma unroll 1
  for (int phase = 0; phase < 2; ++phase) {
#pragma unroll
  for (int i0 = 0; i0 < R; i0 += GR) {
    int64_t e0[GR];
    int32_t cnt[GR];
#pragma unroll
    for (int g = 0; g < GR; ++g) {
      const bool ex = i0 + g < rows;
      const int64_t r = ex ? r0 + i0 + g : r0;
      const int32_t rc = static_cast<int32_t>(r);
      const int32_t blen = (rc + h > n32 - 1 ? n32 - 1 : rc + h) - (rc - h < 0 ? 0 : rc - h) + 1;
      const int64_t rb = ld_rp<RP>(p.row_ptr, r);
      const int32_t nl = __ldg(p.nlow + r);
      e0[g] = phase == 0 ? rb : rb + nl + blen;
      cnt[g] = !ex ? 0 : (phase == 0 ? nl : static_cast<int32_t>(ld_rp<RP>(p.row_ptr, r + 1) - e0[g]));
    }
    offband<F, GR, D>(p, gb, ring, ok, e0, cnt, acc + i0, lane);
  }
  if (phase == 1) break;

  // 2. the band sweep
  auto load_chunk = [&](int32_t m, Val (&regs)[NV]) {
    const int32_t cc = cs + m * KC + kl;
    if (m >= m_lo && m < m_hi) {
#pragma unroll
      for (int j = 0; j < NV; ++j) regs[j] = F::ldp(vp[j] + cc);
    } else {
#pragma unroll
      for (int j = 0; j < NV; ++j) regs[j] = cc >= vlo[j] && cc < vhi[j] ? F::ldp(vp[j] + cc) : zero_val(Val{});
    }
  };
  Val regs[NV];
  load_chunk(0, regs);
  double2 wq[kPF][kCH];
#pragma unroll
  for (int k = 0; k < kPF; ++k)
#pragma unroll
    for (int c = 0; c < kCH; ++c)
      wq[k][c] = ok[c] && cs + k < ce ? ld_nc(gb + static_cast<uint64_t>(cs + k) * p.ldg_b + c * 512)
                                      : make_double2(0.0, 0.0);
  const char* wnext = gb + static_cast<uint64_t>(cs + kPF) * p.ldg_b;  // W row of the next refill
#pragma unroll
  for (int j = 0; j < NV; ++j) sm[j * 32 + lane] = regs[j];
  __syncwarp();
  const int32_t rmh = rr0 - h;
  for (int32_t m = 0; m < n_chunks; ++m) {
    if (m + 1 < n_chunks) load_chunk(m + 1, regs);
    const int32_t c0 = cs + m * KC;
    if (m >= m_lo && m < m_hi) {
      constexpr int UK = KC < 8 ? KC : 8;  // columns per unrolled body (code size: the loop must stay in the instruction cache)
#pragma unroll 1
      for (int k0 = 0; k0 < KC; k0 += UK) {
        const Val* smk = sm + k0;
#pragma unroll
        for (int k = 0; k < UK; ++k) {
          double2 w[kCH];
#pragma unroll
          for (int c = 0; c < kCH; ++c) {
            w[c] = wq[k % kPF][c];
            wq[k % kPF][c] = ld_nc(wnext + c * 512);
          }
          wnext += p.ldg_b;
#pragma unroll
          for (int i = 0; i < R; ++i) {
            const Val a = smk[i * KC + k];
#pragma unroll
            for (int c = 0; c < kCH; ++c) acc[i][c] = F::mac(acc[i][c], a, w[c]);
          }
        }
      }
    } else {
#pragma unroll 1
      for (int k0 = 0; k0 < KC; k0 += kPF) {
#pragma unroll
        for (int k = 0; k < kPF; ++k) {
          const int32_t cc = c0 + k0 + k;
          double2 w[kCH];
#pragma unroll
          for (int c = 0; c < kCH; ++c) {
            w[c] = wq[k][c];
            if (ok[c] && cc + kPF < ce) wq[k][c] = ld_nc(wnext + c * 512);
          }
          wnext += p.ldg_b;
#pragma unroll
          for (int i = 0; i < R; ++i) {
            // column cc is in row (r0 + i)'s band iff r0 + i - h <= cc <= r0 + i + h (cc is a valid
            // column already) and the row exists
            if (static_cast<uint32_t>(cc - rmh - i) <= static_cast<uint32_t>(2 * h) && i < rows && cc < ce) {
              const Val a = sm[i * KC + k0 + k];
#pragma unroll
              for (int c = 0; c < kCH; ++c) acc[i][c] = F::mac(acc[i][c], a, w[c]);
            }
          }
        }
      }
    }
    __syncwarp();
    if (m + 1 < n_chunks) {
#pragma unroll
      for (int j = 0; j < NV; ++j) sm[j * 32 + lane] = regs[j];
    }
    __syncwarp();
  }

  }  // phases

  // 4. epilogue: v = (((s0 aw) + (s1 w)) - v) + (s2 y)   (cheb_filter.cpp:170-171, 176-177)
  const uint64_t pol = policy_evict_first();
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t r = r0 + i;
    if (i >= rows) continue;
#pragma unroll
    for (int c = 0; c < kCH; ++c) {
      if (!ok[c]) continue;
      const uint32_t o = voff + c * 512;
      const double2 own = ld_nc(p.g + static_cast<uint64_t>(r) * p.ldg_b + o);
      const double2 vv = ld_nc(p.vin + static_cast<uint64_t>(r) * p.ldg_b + o);
      const double2 yy = ld_nc(p.yin + static_cast<uint64_t>(r) * p.ldy_b + o);
      double2 res;
      res.x = __dadd_rn(__dsub_rn(__dadd_rn(__dmul_rn(p.s0, acc[i][c].x), __dmul_rn(p.s1, own.x)), vv.x),
                        __dmul_rn(p.s2, yy.x));
      res.y = __dadd_rn(__dsub_rn(__dadd_rn(__dmul_rn(p.s0, acc[i][c].y), __dmul_rn(p.s1, own.y)), vv.y),
                        __dmul_rn(p.s2, yy.y));
      st_hint(p.out + static_cast<uint64_t>(r) * p.ldo_b + o, res, pol);
    }
  }
}

template <class F, int R, int KC, class RP, int NT, int MINB, int GR, int D>
void launch_band(adp_ctx* ctx, BArgs k, int64_t qv) {
  constexpr int NW = NT / 32;
  k.n_blocks = static_cast<int32_t>((k.n + R - 1) / R);
  k.n_panels = static_cast<int32_t>((qv + 32 * kCH - 1) / (32 * kCH));
  k.valid = static_cast<int32_t>(qv);
  const int64_t groups = (static_cast<int64_t>(k.n_blocks) + NW - 1) / NW;
  const int64_t grid = groups * k.n_panels;
  if (grid >= (int64_t{1} << 31)) fail(ADP_ERR_DIMENSION, "cheb_band: too many tasks");
  auto kern = cheb_band_kernel<F, R, KC, RP, NT, MINB, GR, D>;
  constexpr size_t smem = static_cast<size_t>(NW) * BandSlot<F, R, KC, GR, D>::bytes;
  static_assert(smem * MINB <= 200 * 1024, "band kernel shared memory");
  ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  launch_pdl(ctx, kern, dim3(static_cast<unsigned>(grid)), dim3(NT), smem, k);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

}  // namespace

const BandPlan* get_band_plan(adp_csr* a) {
  if (a->band) return a->band.get();
  auto p = std::make_unique<BandPlan>();
  const int64_t n = a->n_rows;
  a->band = std::move(p);
  BandPlan& b = *a->band;
  if (n != a->n_cols || n < 1024 || n >= (int64_t{1} << 31)) return &b;
  // h from the middle row: the run of consecutive columns that contains the diagonal
  const int64_t r = n / 2;
  int64_t e[2];
  if (a->rp64) {
    ADP_CUDA(cudaMemcpy(e, static_cast<const int64_t*>(a->row_ptr) + r, 16, cudaMemcpyDeviceToHost));
  } else {
    int32_t e32[2];
    ADP_CUDA(cudaMemcpy(e32, static_cast<const int32_t*>(a->row_ptr) + r, 8, cudaMemcpyDeviceToHost));
    e[0] = e32[0];
    e[1] = e32[1];
  }
  if (e[1] - e[0] <= 0 || e[1] - e[0] > (1 << 20)) return &b;
  std::vector<int32_t> cols(static_cast<size_t>(e[1] - e[0]));
  ADP_CUDA(cudaMemcpy(cols.data(), a->col_idx + e[0], cols.size() * 4, cudaMemcpyDeviceToHost));
  const auto it = std::find(cols.begin(), cols.end(), static_cast<int32_t>(r));
  if (it == cols.end()) return &b;
  int64_t k0 = it - cols.begin(), k1 = k0;
  while (k0 > 0 && cols[k0 - 1] == cols[k0] - 1) --k0;
  while (k1 + 1 < static_cast<int64_t>(cols.size()) && cols[k1 + 1] == cols[k1] + 1) ++k1;
  const int64_t h = std::min<int64_t>(r - cols[k0], cols[k1] - r);
  if (h < 16) return &b;  // no band worth a sweep
  int* bad = nullptr;
  ADP_CUDA(cudaMalloc(&b.d_nlow, static_cast<size_t>(n) * 4));
  ADP_CUDA(cudaMalloc(&bad, sizeof(int)));
  ADP_CUDA(cudaMemset(bad, 0, sizeof(int)));
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32));
  if (a->rp64)
    band_plan_kernel<int64_t><<<grid, 256>>>(static_cast<const int64_t*>(a->row_ptr), a->col_idx, n, h, b.d_nlow, bad);
  else
    band_plan_kernel<int32_t><<<grid, 256>>>(static_cast<const int32_t*>(a->row_ptr), a->col_idx, n, h, b.d_nlow, bad);
  ADP_LAUNCH_CHECK();
  int hbad = 1;
  ADP_CUDA(cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(bad);
  b.h = h;
  b.valid = hbad == 0;
  return &b;
}

bool launch_step_band(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  const adp_csr* a = s.a;
  if (mode != StepMode::Step) return false;
  if (ctx->variant == 0 && !ctx->auto_band) return false;
  if (ctx->variant != 0 && (ctx->variant < 6 || ctx->variant > 11)) return false;
  if (s.row_begin != 0 || s.row_end != a->n_rows || s.goff != 0 || s.n_push != 0) return false;
  if (a->n_rows != a->n_cols || a->nnz < 32 * a->n_rows) return false;  // long rows only (config 5: 541)
  const bool cplx = a->dtype == ADP_C128;
  const int epv = cplx ? 1 : 2;
  if (s.ld % epv || s.ld_y % epv || s.ld_out % epv) return false;
  for (int64_t ld : {s.ld, s.ld_y, s.ld_out})
    if ((ld / epv) * 16 >= (int64_t{1} << 32)) return false;
  const BandPlan* bp = get_band_plan(const_cast<adp_csr*>(a));
  if (!bp->valid) return false;
  BArgs k{};
  k.row_ptr = a->row_ptr;
  k.col = a->col_idx;
  k.val = a->values;
  k.nlow = bp->d_nlow;
  k.g = static_cast<const char*>(s.gsrc);
  k.vin = static_cast<const char*>(s.vin);
  k.yin = static_cast<const char*>(s.yin);
  k.out = static_cast<char*>(s.out);
  k.ldg_b = static_cast<uint32_t>((s.ld / epv) * 16);
  k.ldy_b = static_cast<uint32_t>((s.ld_y / epv) * 16);
  k.ldo_b = static_cast<uint32_t>((s.ld_out / epv) * 16);
  k.n = a->n_rows;
  k.h = static_cast<int32_t>(bp->h);
  k.s0 = s.s0;
  k.s1 = s.s1;
  k.s2 = s.s2;
  const int64_t qv = (s.q + epv - 1) / epv;
  // geometry (rows per warp R, columns per value chunk KC, threads per CTA, CTAs per SM); the automatic
  // choice is variant 6's, variants 7-11 are measurement alternatives
#define ADP_BAND(R_, KC_, NT_, MB_, GR_, D_)                                                                     \
  do {                                                                                                           \
    if (cplx) a->rp64 ? launch_band<CplxB, R_, KC_, int64_t, NT_, MB_, GR_, D_>(ctx, k, qv)                       \
                      : launch_band<CplxB, R_, KC_, int32_t, NT_, MB_, GR_, D_>(ctx, k, qv);                      \
    else a->rp64 ? launch_band<RealB, R_, KC_, int64_t, NT_, MB_, GR_, D_>(ctx, k, qv)                            \
                 : launch_band<RealB, R_, KC_, int32_t, NT_, MB_, GR_, D_>(ctx, k, qv);                           \
  } while (0)
  switch (ctx->variant) {
    case 7: ADP_BAND(4, 32, 256, 2, 4, 2); break;
    case 8: ADP_BAND(4, 32, 256, 2, 2, 4); break;
    case 9: ADP_BAND(6, 16, 256, 2, 3, 2); break;
    case 10: ADP_BAND(4, 32, 256, 2, 4, 3); break;
    case 11: ADP_BAND(8, 16, 128, 3, 4, 2); break;
    default: ADP_BAND(8, 16, 192, 2, 4, 2); break;
  }
#undef ADP_BAND
  return true;
}

}  // namespace adp
