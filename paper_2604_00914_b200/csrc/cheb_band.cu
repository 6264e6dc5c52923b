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
// (row by row, before the sweep), its band (during the sweep, column ascending), its upper off-band
// entries (after it) -- which is CSR order, so the result is bitwise the lean kernel's (complex: four
// DFMA per entry, the order the complex path defines; real: the reference's unfused mul + add).
//
// The host derives h from the middle row and a device kernel verifies, for EVERY row, that its
// columns are [lower off-band | max(0, r - h) .. min(n - 1, r + h) | upper off-band] and records
// the number of lower entries (BandPlan, once per operator: config 5's 43 GB operator is generated
// on the device and is never copied to the host for this).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
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
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};
struct CplxB {
  using Val = double2;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double2*>(p) + k); }
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

// One warp per (block of R consecutive rows, panel of 32 x CH 16-byte vectors); Step mode.
template <class F, int R, int CH, class RP, int MINB>
__global__ void __launch_bounds__(256, MINB) cheb_band_kernel(const BArgs p) {
  const int lane = threadIdx.x & 31;
  const int64_t task = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (task >= static_cast<int64_t>(p.n_blocks) * p.n_panels) return;  // warp-uniform
  const int panel = static_cast<int>(task / p.n_blocks);
  const int64_t r0 = (task - static_cast<int64_t>(panel) * p.n_blocks) * R;
  const uint32_t voff = (static_cast<uint32_t>(panel) * 32 * CH + lane) * 16u;
  bool ok[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) ok[c] = panel * 32 * CH + c * 32 + lane < p.valid;
  // row metadata (the operator is constant: read before the wait): band start entry, first band
  // column and band length of each row
  int64_t bs[R];
  int32_t b0[R], blen[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t r = r0 + i < p.n ? r0 + i : p.n - 1;
    bs[i] = ld_rp<RP>(p.row_ptr, r) + __ldg(p.nlow + r);
    const int64_t lo = r - p.h < 0 ? 0 : r - p.h, hi = r + p.h > p.n - 1 ? p.n - 1 : r + p.h;
    b0[i] = static_cast<int32_t>(lo);
    blen[i] = r0 + i < p.n ? static_cast<int32_t>(hi - lo + 1) : 0;
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const char* gb = p.g + voff;
  double2 acc[R][CH];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[i][c] = make_double2(0.0, 0.0);

  // 1. lower off-band entries, row by row (they precede the band in every row's column order)
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (r0 + i >= p.n) continue;
    for (int64_t e = ld_rp<RP>(p.row_ptr, r0 + i); e < bs[i]; ++e) {
      const char* src = gb + static_cast<uint64_t>(__ldg(p.col + e)) * p.ldg_b;
      const typename F::Val v = F::load(p.val, e);
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if (ok[c]) acc[i][c] = F::mac(acc[i][c], v, ld_nc(src + c * 512));
    }
  }
  // 2. the band sweep: columns of the union of the R bands, ascending; each W row panel is loaded
  // once (PF columns ahead) and applied to every row whose band holds the column
  const int32_t cs = b0[0];
  int32_t ce = b0[0] + blen[0];
#pragma unroll
  for (int i = 1; i < R; ++i) ce = blen[i] ? b0[i] + blen[i] : ce;
  constexpr int PF = 2;
  double2 wq[PF][CH];
#pragma unroll
  for (int k = 0; k < PF; ++k)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      wq[k][c] = ok[c] && cs + k < ce ? ld_nc(gb + static_cast<uint64_t>(cs + k) * p.ldg_b + c * 512)
                                      : make_double2(0.0, 0.0);
  for (int32_t col = cs; col < ce; col += PF) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int32_t cc = col + k;
      if (cc >= ce) break;
      double2 w[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        w[c] = wq[k][c];
        if (ok[c] && cc + PF < ce) wq[k][c] = ld_nc(gb + static_cast<uint64_t>(cc + PF) * p.ldg_b + c * 512);
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int32_t d = cc - b0[i];
        if (static_cast<uint32_t>(d) < static_cast<uint32_t>(blen[i])) {
          const typename F::Val v = F::load(p.val, bs[i] + d);
#pragma unroll
          for (int c = 0; c < CH; ++c) acc[i][c] = F::mac(acc[i][c], v, w[c]);
        }
      }
    }
  }
  // 3. upper off-band entries, row by row
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (r0 + i >= p.n) continue;
    const int64_t e1 = ld_rp<RP>(p.row_ptr, r0 + i + 1);
    for (int64_t e = bs[i] + blen[i]; e < e1; ++e) {
      const char* src = gb + static_cast<uint64_t>(__ldg(p.col + e)) * p.ldg_b;
      const typename F::Val v = F::load(p.val, e);
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if (ok[c]) acc[i][c] = F::mac(acc[i][c], v, ld_nc(src + c * 512));
    }
  }
  // 4. epilogue: v = (((s0 aw) + (s1 w)) - v) + (s2 y)   (cheb_filter.cpp:170-171, 176-177)
  const uint64_t pol = policy_evict_first();
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t r = r0 + i;
    if (r >= p.n) continue;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
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

template <class F, int R, int CH, class RP, int MINB>
void launch_band(adp_ctx* ctx, BArgs k, int64_t qv) {
  k.n_blocks = static_cast<int32_t>((k.n + R - 1) / R);
  k.n_panels = static_cast<int32_t>((qv + 32 * CH - 1) / (32 * CH));
  k.valid = static_cast<int32_t>(qv);
  const int64_t tasks = static_cast<int64_t>(k.n_blocks) * k.n_panels;
  const int64_t grid = (tasks + 7) / 8;
  if (grid >= (int64_t{1} << 31)) fail(ADP_ERR_DIMENSION, "cheb_band: too many tasks");
  launch_pdl(ctx, cheb_band_kernel<F, R, CH, RP, MINB>, dim3(static_cast<unsigned>(grid)), dim3(256), 0, k);
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
  if (ctx->variant != 0 && ctx->variant != 6 && ctx->variant != 7) return false;
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
  if (ctx->variant == 7) {  // measurement: 4-row blocks (fewer registers, more resident warps)
    if (cplx) a->rp64 ? launch_band<CplxB, 4, 2, int64_t, 2>(ctx, k, qv) : launch_band<CplxB, 4, 2, int32_t, 2>(ctx, k, qv);
    else a->rp64 ? launch_band<RealB, 4, 2, int64_t, 2>(ctx, k, qv) : launch_band<RealB, 4, 2, int32_t, 2>(ctx, k, qv);
  } else if (cplx) {
    if (a->rp64) launch_band<CplxB, 8, 2, int64_t, 1>(ctx, k, qv);
    else launch_band<CplxB, 8, 2, int32_t, 1>(ctx, k, qv);
  } else {
    if (a->rp64) launch_band<RealB, 8, 2, int64_t, 1>(ctx, k, qv);
    else launch_band<RealB, 8, 2, int32_t, 1>(ctx, k, qv);
  }
  return true;
}

}  // namespace adp
