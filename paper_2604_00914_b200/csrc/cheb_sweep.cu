// Fused Clenshaw step for constant-coefficient 3-D stencil operators: the
// plane-sweep ("sweep") kernel, sm_100a.
//
// One degree step of clenshaw_apply (proj/src/cheb_filter.cpp:167-177: maspmm,
// tiled_matrix.hpp:184-210, fused with the recurrence update) on an operator
// that IS a radius-1 stencil on a structured grid -- configs 2 and 4: a 7-point
// or 27-point Laplacian whose off-diagonal values are one constant per offset,
// plus a per-row diagonal (the potential). The host verifies that property
// entry by entry against the CSR (StencilPlan, once per operator) and keeps the
// 26 constants as kernel parameters and the diagonal as one array, so the
// operator costs 8 B per row instead of 12 B per nonzero -- and, because it is
// that cheap, column panels can be narrow (32 fp64 columns, 256 B per row).
//
// Narrow panels make a 2.5-D blocking possible: a CTA owns a TX x TY tile of
// grid points (8 x 8) and one panel, and sweeps the tile through all z planes.
// Per plane z, ONE 4-D TMA box brings W's (TX+2) x (TY+2) halo tile into shared
// memory (grid edges: TMA's zero fill), and every W value is read from shared
// memory by the nine rows of each of the three planes z-1, z, z+1 it feeds:
// each output point keeps three accumulators (planes z+1, z, z-1) in
// registers, plane z's products are added to all three, and plane z-1 is
// complete -- it takes its epilogue (V and Y tiles, TMA, L2 evict-first) and is
// stored. W crosses L2 -> SM (TX+2)(TY+2)/(TX TY) = 1.56 times instead of 27
// (lean) or 8 (cube) gathered rows per row; DRAM reads W once (neighbouring
// tiles of a panel sweep the same planes at the same time, and one plane of a
// panel is 4 MB of L2 on config 4).
//
// Bitwise equal to the CSR kernels: every output accumulates its products from
// +0 in ascending column order ((dz, dy, dx) lexicographic: plane z-1's nine,
// plane z's nine, plane z+1's nine -- the planes arrive in that order), with
// unfused __dmul_rn / __dadd_rn and the reference's epilogue expression. Grid
// points outside the grid read W = +0 from TMA's fill: v * 0 = +-0, and
// acc + (+-0) == acc for every acc the sum can reach (it starts at +0 and a
// round-to-nearest sum is never -0 unless both terms are), so the missing CSR
// entries of boundary rows are bitwise no-ops. The plan requires finite values.
//
// Warp roles: NW consumer warps (warp w owns tile row y0 + w, lane = column of
// the panel, kTX points along x per thread) and one producer warp whose lane 0
// issues the TMA copies into two rings (W + diagonal per plane; V + Y per
// output plane), with full / empty mbarriers. The grid is persistent (one CTA
// per SM: ~200 KB of shared memory) and walks (panel, tile) items panel-major.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

StencilPlan::~StencilPlan() { cudaFree(d_diag); }

namespace {

// ---- stencil detection (host, once per operator) -----------------------------------------
struct Off {
  int dx, dy, dz;
};

// Row r of the operator is grid point g = r + goff of an extended grid whose points are the operator's
// columns (goff != 0: a rank's rows of the row partition, columns in its halo-extended local layout).
void build_stencil_plan(adp_csr* a, int64_t goff, StencilPlan& p) {
  const int64_t n = a->n_rows, nc = a->n_cols;
  p.goff = goff;
  if (a->dtype != ADP_F64) return void(p.why = "not real fp64");
  if (n < 8 || nc >= (int64_t{1} << 31) || goff < 0 || goff + n > nc) return void(p.why = "shape");
  if (a->nnz > 27 * n || a->nnz < 2 * n) return void(p.why = "row lengths");
  ensure_host_copy(a);
  const std::vector<int64_t>& rp = a->h_row_ptr;
  const std::vector<int32_t>& ci = a->h_col;
  const double* val = static_cast<const double*>(a->h_values);
  // the longest row holds the whole offset set
  int64_t kmax = 0, rmax = 0;
  for (int64_t r = 0; r < n; ++r)
    if (rp[r + 1] - rp[r] > kmax) kmax = rp[r + 1] - rp[r], rmax = r;
  if (kmax != 27 && kmax != 7) return void(p.why = "longest row is not 7 or 27 entries");
  std::vector<int64_t> off(static_cast<size_t>(kmax));
  for (int64_t k = 0; k < kmax; ++k) off[k] = static_cast<int64_t>(ci[rp[rmax] + k]) - (rmax + goff);
  // runs of consecutive offsets and their centres
  std::vector<int64_t> centre, len;
  for (int64_t k = 0; k < kmax;) {
    int64_t m = 1;
    while (k + m < kmax && off[k + m] == off[k + m - 1] + 1) ++m;
    if (m != 1 && m != 3) return void(p.why = "offset runs");
    centre.push_back(off[k] + (m == 3 ? 1 : 0));
    len.push_back(m);
    k += m;
  }
  int64_t sy = 0, sz = 0;
  if (kmax == 27) {
    if (centre.size() != 9) return void(p.why = "27 entries but not 9 runs of 3");
    sy = centre[5];
    sz = centre[7];
  } else {
    if (centre.size() != 5 || len[0] != 1 || len[1] != 1 || len[2] != 3 || len[3] != 1 || len[4] != 1)
      return void(p.why = "7 entries but not a star");
    sy = centre[3];
    sz = centre[4];
  }
  const int64_t h = static_cast<int64_t>(centre.size()) / 2;
  for (int64_t j = 0; j <= h; ++j)
    if (centre[h - j] != -centre[h + j]) return void(p.why = "offsets not symmetric");
  if (sy < 3 || sz <= sy || sz % sy != 0 || nc % sz != 0 || n % sz != 0 || goff % sz != 0)
    return void(p.why = "no grid strides (or rows / offset not whole planes)");
  p.nx = sy;
  p.ny = sz / sy;
  p.nz = n / sz;    // planes of the operator's rows
  p.nzw = nc / sz;  // planes of the (extended) grid its columns index
  if (p.ny < 3) return void(p.why = "grid too thin");
  p.kind = static_cast<int>(kmax);
  // the offset set in ascending column order: (dz, dy, dx) lexicographic
  std::vector<Off> set;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int m = (dx != 0) + (dy != 0) + (dz != 0);
        if (p.kind == 27 || m <= 1) set.push_back({dx, dy, dz});
      }
  // verify every row: columns exactly the in-grid offsets in order, values constant per
  // offset (bitwise), the centre per row, all finite
  p.nxp = (p.nx + 1) / 2 * 2;
  std::vector<double> diag(static_cast<size_t>(p.nz * p.ny * p.nxp), 0.0);
  bool have[27] = {};
  for (int64_t r = 0; r < n; ++r) {
    const int64_t g = r + goff;
    const int64_t x = g % p.nx, y = (g / p.nx) % p.ny, z = g / sz;
    int64_t e = rp[r];
    const int64_t e1 = rp[r + 1];
    for (const Off& o : set) {
      if (x + o.dx < 0 || x + o.dx >= p.nx || y + o.dy < 0 || y + o.dy >= p.ny || z + o.dz < 0 || z + o.dz >= p.nzw)
        continue;
      const int64_t c = g + o.dx + sy * o.dy + sz * o.dz;
      if (e >= e1 || ci[e] != c) return void(p.why = "row " + std::to_string(r) + ": pattern");
      const double v = val[e];
      if (!std::isfinite(v)) return void(p.why = "non-finite value");
      const int idx = (o.dz + 1) * 9 + (o.dy + 1) * 3 + (o.dx + 1);
      if (idx == 13) {
        diag[static_cast<size_t>(((r / sz) * p.ny + y) * p.nxp + x)] = v;
      } else if (!have[idx]) {
        p.w[idx] = v;
        have[idx] = true;
      } else if (std::memcmp(&v, &p.w[idx], sizeof v) != 0) {
        return void(p.why = "off-diagonal values vary");
      }
      ++e;
    }
    if (e != e1) return void(p.why = "row " + std::to_string(r) + ": extra entries");
  }
  // shared class products: 27-point weights that depend only on the distance class m (bitwise equal
  // within a class); 7-point neighbour weights all exactly -1
  auto same = [](double u, double v) { return std::memcmp(&u, &v, sizeof u) == 0; };
  p.classes = true;
  bool seen[4] = {};
  for (const Off& o : set) {
    const int idx = (o.dz + 1) * 9 + (o.dy + 1) * 3 + (o.dx + 1);
    const int m = std::abs(o.dx) + std::abs(o.dy) + std::abs(o.dz);
    if (m == 0) continue;
    if (!have[idx]) p.classes = false;  // an offset no row holds: keep the general path
    if (p.kind == 7 && !same(p.w[idx], -1.0)) p.classes = false;
    if (p.kind == 27) {
      if (!seen[m]) p.cls[m] = p.w[idx], seen[m] = true;
      if (!same(p.cls[m], p.w[idx])) p.classes = false;
    }
  }
  ADP_CUDA(cudaMalloc(&p.d_diag, diag.size() * sizeof(double)));
  ADP_CUDA(cudaMemcpy(p.d_diag, diag.data(), diag.size() * sizeof(double), cudaMemcpyHostToDevice));
  plan_uploads_done();
  p.valid = true;
}

// ---- device helpers -----------------------------------------------------------------------
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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
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
// 4-D / 3-D TMA tile loads (box from the tensor map; coordinates outside the tensor read as +0)
__device__ __forceinline__ void tma4d(void* dst, const CUtensorMap* tm, int32_t c0, int32_t c1, int32_t c2, int32_t c3,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma4d_hint(void* dst, const CUtensorMap* tm, int32_t c0, int32_t c1, int32_t c2,
                                           int32_t c3, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4, %5}], [%6], %7;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* tm, int32_t c0, int32_t c1, int32_t c2,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void st_hint(void* ptr, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(ptr), "d"(v), "l"(pol) : "memory");
}
// Product arithmetic of the sweep kernel, all the reference's unfused SSE2 rounding: kExact: every
// product rounded then added; kShared: the same, with each distance-class product formed once per
// loaded W value; kUnitNeg: the 7-point star with all neighbour weights -1 (subtractions). (A DFMA
// variant measured the same sustained time once the product count was shared: not kept.)
constexpr int kExact = 0, kShared = 1, kUnitNeg = 2;
template <int ARITH>
__device__ __forceinline__ double mac(double acc, double v, double w) {
  return __dadd_rn(acc, __dmul_rn(v, w));
}

// ---- the kernel -----------------------------------------------------------------------------
constexpr int kTX = 8;   // grid points per thread along x
constexpr int kPW = 32;  // fp64 columns per panel (one per lane)
constexpr int kSW = 4;   // W ring stages (planes z-1 and z held, two ahead)
constexpr int kSV = 3;   // V / Y ring stages

template <int NW>
struct Geo {
  static constexpr int WX = kTX + 2, WY = NW + 2;
  static constexpr uint32_t kW = WX * WY * kPW * 8;                    // W halo tile of one plane
  static constexpr uint32_t kD = kTX * NW * 8;                         // the tile's centre values
  static constexpr uint32_t kWS = (kW + kD + 127) / 128 * 128;         // one W stage
  static constexpr uint32_t kT = kTX * NW * kPW * 8;                   // one V (or Y) tile
  static constexpr uint32_t kVS = 2 * kT;                              // one V / Y stage
  static constexpr uint32_t kBar = kSW * kWS + kSV * kVS;              // the mbarriers
  static constexpr uint32_t kSmem = kBar + 2 * (kSW + kSV) * 8;
};

struct SwArgs {
  char* out;
  uint64_t ldo_b;
  int32_t nx, ny, q;
  int32_t nzo;       // output planes of the launch
  int32_t zv0;       // V / Y / out / diagonal plane of output plane 0 (row_begin / plane)
  int32_t zw0;       // W plane of output plane 0 ((row_begin + goff) / plane)
  int32_t wlo, whi;  // W planes the launch reads: [zw0 - 1, zw0 + nzo] inside the tensor
  int32_t nzv;       // planes of the V / Y / diagonal tensors
  int32_t tiles_x, tiles_y, n_items;
  double s0, s1, s2;
  double w[27];  // constant values by offset; read as constant-bank operands of the DMULs
  double c[4];   // kShared: the value of distance class m = |dx| + |dy| + |dz| (m = 1..3)
  // peer-memory halo (multi-GPU row partition): output rows r in [lo, hi) are also stored to
  // dst + (r + shift) * ld_b, a neighbour's halo rows mapped over NVLink (see cheb_lean.cu)
  PushTarget push[kMaxPush];
  int32_t n_push;
};

template <int NW, int KIND, int ARITH, bool PUSH>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    cheb_sweep_kernel(const __grid_constant__ SwArgs p, const __grid_constant__ CUtensorMap tm_w,
                      const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ CUtensorMap tm_v,
                      const __grid_constant__ CUtensorMap tm_y) {
  using G = Geo<NW>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full_w = reinterpret_cast<uint64_t*>(smem + G::kBar);
  uint64_t* empty_w = full_w + kSW;
  uint64_t* full_v = empty_w + kSW;
  uint64_t* empty_v = full_v + kSV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSW; ++i) {
      mbar_init(full_w + i, 1);
      mbar_init(empty_w + i, NW);
    }
    for (int i = 0; i < kSV; ++i) {
      mbar_init(full_v + i, 1);
      mbar_init(empty_v + i, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // PDL: nothing the previous degree step writes is touched before this
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int tiles = p.tiles_x * p.tiles_y;

  if (warp == NW) {  // producer: per W plane its halo tile + the centre values of that plane's outputs,
                     // then the V / Y tiles of that output plane (consumed one plane later)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first(1.0f);
      uint32_t sw = 0, pw = 1, sv = 0, pv = 1;  // a fresh empty barrier's preceding phase counts as done
      for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
        const int panel = item / tiles, t = item - panel * tiles;
        const int ty = t / p.tiles_x, tx = t - ty * p.tiles_x;
        const int x0 = tx * kTX, y0 = ty * NW, c0 = panel * kPW;
        for (int wz = p.wlo; wz <= p.whi; ++wz) {
          const int o = wz - p.zw0;  // the output plane whose own W plane this is
          mbar_wait(empty_w + sw, pw);
          uint8_t* ws = smem + sw * G::kWS;
          mbar_expect_tx(full_w + sw, G::kW + G::kD);
          tma4d(ws, &tm_w, c0, x0 - 1, y0 - 1, wz, full_w + sw);
          tma3d(ws + G::kW, &tm_d, x0, y0, min(max(p.zv0 + o, 0), p.nzv - 1), full_w + sw);  // unused unless o is an output
          if (++sw == kSW) sw = 0, pw ^= 1;
          if (o >= 0 && o < p.nzo) {
            mbar_wait(empty_v + sv, pv);
            uint8_t* vs = smem + kSW * G::kWS + sv * G::kVS;
            mbar_expect_tx(full_v + sv, G::kVS);
            tma4d_hint(vs, &tm_v, c0, x0, y0, p.zv0 + o, full_v + sv, pol);
            tma4d_hint(vs + G::kT, &tm_y, c0, x0, y0, p.zv0 + o, full_v + sv, pol);
            if (++sv == kSV) sv = 0, pv ^= 1;
          }
        }
      }
    }
    return;
  }

  // consumers: warp = tile row, lane = panel column, kTX points along x
  const int yl = warp;
  const uint64_t pol = policy_evict_first(1.0f);
  uint32_t sw = 0, pw = 0, sv = 0, pv = 0, sprev = 0;
  bool have_prev = false;
  double A0[kTX], A1[kTX], A2[kTX];
#pragma unroll
  for (int x = 0; x < kTX; ++x) A0[x] = A1[x] = A2[x] = 0.0;

  for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
    const int panel = item / tiles, t = item - panel * tiles;
    const int ty = t / p.tiles_x, tx = t - ty * p.tiles_x;
    const int x0 = tx * kTX, y = ty * NW + yl, c = panel * kPW + lane;
    const bool live = y < p.ny && c < p.q;
    char* obase = p.out + static_cast<uint64_t>(c) * 8;

    // one step per W plane wz (and one after the last): plane wz's products into lo (the output whose own
    // plane is wz - 1), mid (wz), hi (wz + 1); then lo's epilogue if it is an output plane of the launch
    auto step = [&](int wz, double(&lo)[kTX], double(&mid)[kTX], double(&hi)[kTX]) {
      const bool real = wz <= p.whi;
      if (real) {
        mbar_wait(full_w + sw, pw);
        const double* ws = reinterpret_cast<const double*>(smem + sw * G::kWS);
        const double* ds = reinterpret_cast<const double*>(smem + sw * G::kWS + G::kW) + yl * kTX;
        if constexpr (KIND == 27 && ARITH == kShared) {
          // weights depend only on m = |dx| + |dy| + |dz| (c1 faces, c2 edges, c3 corners): each loaded W
          // value's products c_m * w are rounded ONCE and added by every output that holds it at class m
          // -- the same rounded product the reference forms per entry, so the sums are bitwise its own
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) {
            double w[kTX + 2], p1[kTX + 2], p2[kTX + 2], p3[kTX + 2];
            const double* row = ws + (yl + dy) * G::WX * kPW + lane;
#pragma unroll
            for (int i = 0; i < kTX + 2; ++i) {
              w[i] = row[i * kPW];
              p1[i] = __dmul_rn(p.c[1], w[i]);
              p2[i] = __dmul_rn(p.c[2], w[i]);
              if (dy != 1) p3[i] = __dmul_rn(p.c[3], w[i]);
            }
#pragma unroll
            for (int x = 0; x < kTX; ++x) {
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
                const int i = x + dx, m = (dx != 1) + (dy != 1);  // in-plane distance class
                const double pz = m == 0 ? p1[i] : (m == 1 ? p2[i] : p3[i]);  // class m + 1 (dz = -1, +1)
                hi[x] = __dadd_rn(hi[x], pz);
                mid[x] = __dadd_rn(mid[x], m == 0 ? __dmul_rn(ds[x], w[i]) : (m == 1 ? p1[i] : p2[i]));
                lo[x] = __dadd_rn(lo[x], pz);
              }
            }
          }
        } else if constexpr (KIND == 27) {
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) {
            double w[kTX + 2];
            const double* row = ws + (yl + dy) * G::WX * kPW + lane;
#pragma unroll
            for (int i = 0; i < kTX + 2; ++i) w[i] = row[i * kPW];
#pragma unroll
            for (int x = 0; x < kTX; ++x) {
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
                const double wv = w[x + dx];
                hi[x] = mac<ARITH>(hi[x], p.w[dy * 3 + dx], wv);  // dz = -1 entries of plane wz+1
                mid[x] = mac<ARITH>(mid[x], (dy == 1 && dx == 1) ? ds[x] : p.w[9 + dy * 3 + dx], wv);
                lo[x] = mac<ARITH>(lo[x], p.w[18 + dy * 3 + dx], wv);  // dz = +1 entries of plane wz-1
              }
            }
          }
        } else {  // 7-point star: (0,0,-1) (0,-1,0) (-1,0,0) centre (1,0,0) (0,1,0) (0,0,1)
          const double* up = ws + yl * G::WX * kPW + lane;
          const double* ce = up + G::WX * kPW;
          const double* dn = ce + G::WX * kPW;
          double w[kTX + 2];
#pragma unroll
          for (int i = 0; i < kTX + 2; ++i) w[i] = ce[i * kPW];
          if constexpr (ARITH == kUnitNeg) {
            // every neighbour weight is exactly -1: acc + (-1 * w) == acc - w bitwise (IEEE x - y = x + (-y))
#pragma unroll
            for (int x = 0; x < kTX; ++x) {
              hi[x] = __dsub_rn(hi[x], w[x + 1]);
              mid[x] = __dsub_rn(mid[x], up[(x + 1) * kPW]);
              mid[x] = __dsub_rn(mid[x], w[x]);
              mid[x] = __dadd_rn(mid[x], __dmul_rn(ds[x], w[x + 1]));
              mid[x] = __dsub_rn(mid[x], w[x + 2]);
              mid[x] = __dsub_rn(mid[x], dn[(x + 1) * kPW]);
              lo[x] = __dsub_rn(lo[x], w[x + 1]);
            }
          } else {
#pragma unroll
            for (int x = 0; x < kTX; ++x) {
              hi[x] = mac<ARITH>(hi[x], p.w[4], w[x + 1]);
              mid[x] = mac<ARITH>(mid[x], p.w[10], up[(x + 1) * kPW]);
              mid[x] = mac<ARITH>(mid[x], p.w[12], w[x]);
              mid[x] = mac<ARITH>(mid[x], ds[x], w[x + 1]);
              mid[x] = mac<ARITH>(mid[x], p.w[14], w[x + 2]);
              mid[x] = mac<ARITH>(mid[x], p.w[16], dn[(x + 1) * kPW]);
              lo[x] = mac<ARITH>(lo[x], p.w[22], w[x + 1]);
            }
          }
        }
      }
      const int o = wz - p.zw0 - 1;
      if (o >= 0 && o < p.nzo) {  // complete: v = (((s0 aw) + (s1 w)) - v) + (s2 y)  (cheb_filter.cpp:170-171,176-177)
        mbar_wait(full_v + sv, pv);
        const double* own = reinterpret_cast<const double*>(smem + sprev * G::kWS) + ((yl + 1) * G::WX + 1) * kPW + lane;
        const double* vs = reinterpret_cast<const double*>(smem + kSW * G::kWS + sv * G::kVS) + yl * kTX * kPW + lane;
        const double* ys = vs + kTX * NW * kPW;
        if (live) {
          const int64_t rrow = (static_cast<int64_t>(p.zv0 + o) * p.ny + y) * p.nx + x0;  // operator row of x = 0
          char* ob = obase + static_cast<uint64_t>(rrow) * p.ldo_b;
#pragma unroll
          for (int x = 0; x < kTX; ++x) {
            if (x0 + x < p.nx) {
              const double res =
                  __dadd_rn(__dsub_rn(__dadd_rn(__dmul_rn(p.s0, lo[x]), __dmul_rn(p.s1, own[x * kPW])), vs[x * kPW]),
                            __dmul_rn(p.s2, ys[x * kPW]));
              st_hint(ob + static_cast<uint64_t>(x) * p.ldo_b, res, pol);
              if constexpr (PUSH) {  // rows a neighbour needs, also into its halo (peer memory over NVLink)
                for (int tgt = 0; tgt < p.n_push; ++tgt) {
                  const int64_t r = rrow + x;
                  if (r >= p.push[tgt].lo && r < p.push[tgt].hi)
                    *reinterpret_cast<double*>(p.push[tgt].dst + static_cast<uint64_t>(r + p.push[tgt].shift) *
                                                                     p.push[tgt].ld_b + static_cast<uint64_t>(c) * 8) = res;
                }
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_v + sv);
        if (++sv == kSV) sv = 0, pv ^= 1;
      }
      if (have_prev) {  // plane wz - 1 is read for the last time (own rows of lo's epilogue)
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_w + sprev);
      }
#pragma unroll
      for (int x = 0; x < kTX; ++x) lo[x] = 0.0;  // becomes plane wz+2's accumulator
      have_prev = real;
      if (real) {
        sprev = sw;
        if (++sw == kSW) sw = 0, pw ^= 1;
      }
    };

    for (int wz = p.wlo;;) {
      step(wz, A2, A0, A1);
      if (++wz > p.whi + 1) break;
      step(wz, A0, A1, A2);
      if (++wz > p.whi + 1) break;
      step(wz, A1, A2, A0);
      if (++wz > p.whi + 1) break;
    }
    // the roles rotate with wz; the next item starts again with (A2, A0, A1), all zero (accumulators of
    // planes past the launch's outputs hold products that no output takes: cleared)
#pragma unroll
    for (int x = 0; x < kTX; ++x) A0[x] = A1[x] = A2[x] = 0.0;
  }
  if (PUSH) __threadfence_system();  // the peer stores are performed before the signal kernel that follows
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

CUtensorMap make_map(int rank, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                     const cuuint32_t* box) {
  auto enc = encoder();
  if (!enc) fail(ADP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, static_cast<cuuint32_t>(rank), const_cast<void*>(base),
                         dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ADP_ERR_CUDA, "cuTensorMapEncodeTiled (sweep) failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

// A row-major block (row pitch ld_b bytes) of `planes` grid planes seen as [planes][ny][nx][q].
CUtensorMap block_map(const void* base, const StencilPlan& sp, int64_t planes, int64_t q, int64_t ld_b, int bx, int by) {
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(q), static_cast<cuuint64_t>(sp.nx),
                              static_cast<cuuint64_t>(sp.ny), static_cast<cuuint64_t>(planes)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld_b), static_cast<cuuint64_t>(ld_b * sp.nx),
                                 static_cast<cuuint64_t>(ld_b * sp.nx * sp.ny)};
  const cuuint32_t box[4] = {kPW, static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(by), 1};
  return make_map(4, base, dims, strides, box);
}

template <int NW, int KIND, int ARITH, bool PUSH = false>
void launch_sweep(adp_ctx* ctx, const StepArgs& s, const StencilPlan& sp) {
  using G = Geo<NW>;
  const int64_t plane = sp.nx * sp.ny;
  SwArgs k{};
  k.out = static_cast<char*>(s.out);
  k.ldo_b = static_cast<uint64_t>(s.ld_out) * 8;
  k.nx = static_cast<int32_t>(sp.nx);
  k.ny = static_cast<int32_t>(sp.ny);
  k.q = static_cast<int32_t>(s.q);
  k.nzo = static_cast<int32_t>((s.row_end - s.row_begin) / plane);
  k.zv0 = static_cast<int32_t>(s.row_begin / plane);
  k.zw0 = static_cast<int32_t>((s.row_begin + sp.goff) / plane);
  k.wlo = std::max(k.zw0 - 1, 0);
  k.whi = static_cast<int32_t>(std::min<int64_t>(k.zw0 + k.nzo, sp.nzw - 1));
  k.nzv = static_cast<int32_t>(sp.nz);
  k.tiles_x = static_cast<int32_t>((sp.nx + kTX - 1) / kTX);
  k.tiles_y = static_cast<int32_t>((sp.ny + NW - 1) / NW);
  const int64_t panels = (s.q + kPW - 1) / kPW;
  k.n_items = static_cast<int32_t>(panels * k.tiles_x * k.tiles_y);
  k.s0 = s.s0;
  k.s1 = s.s1;
  k.s2 = s.s2;
  for (int i = 0; i < 27; ++i) k.w[i] = sp.w[i];
  for (int i = 0; i < 4; ++i) k.c[i] = sp.cls[i];
  k.n_push = s.n_push;
  for (int t = 0; t < s.n_push; ++t) k.push[t] = s.push[t];
  const CUtensorMap tm_w = block_map(s.gsrc, sp, sp.nzw, s.q, s.ld * 8, kTX + 2, NW + 2);
  const CUtensorMap tm_v = block_map(s.vin, sp, sp.nz, s.q, s.ld * 8, kTX, NW);
  const CUtensorMap tm_y = block_map(s.yin, sp, sp.nz, s.q, s.ld_y * 8, kTX, NW);
  const cuuint64_t ddims[3] = {static_cast<cuuint64_t>(sp.nx), static_cast<cuuint64_t>(sp.ny),
                               static_cast<cuuint64_t>(sp.nz)};
  const cuuint64_t dstr[2] = {static_cast<cuuint64_t>(sp.nxp * 8), static_cast<cuuint64_t>(sp.nxp * sp.ny * 8)};
  const cuuint32_t dbox[3] = {kTX, NW, 1};
  const CUtensorMap tm_d = make_map(3, sp.d_diag, ddims, dstr, dbox);
  auto kern = cheb_sweep_kernel<NW, KIND, ARITH, PUSH>;
  static_assert(G::kSmem <= 227 * 1024, "sweep kernel shared memory");
  ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(G::kSmem)));
  const int grid = static_cast<int>(std::min<int64_t>(k.n_items, ctx->sm_count));
  launch_pdl(ctx, kern, dim3(grid), dim3((NW + 1) * 32), G::kSmem, k, tm_w, tm_d, tm_v, tm_y);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

}  // namespace

const StencilPlan* get_stencil_plan(adp_csr* a, int64_t goff) {
  if (!a->stencil || a->stencil->goff != goff) {
    auto p = std::make_unique<StencilPlan>();
    build_stencil_plan(a, goff, *p);
    a->stencil = std::move(p);
  }
  return a->stencil.get();
}

bool launch_step_sweep(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  const adp_csr* a = s.a;
  if (mode != StepMode::Step || a->dtype != ADP_F64) return false;
  if (ctx->variant == 0 && !ctx->auto_sweep) return false;
  if (ctx->variant != 0 && ctx->variant != 5) return false;
  if (a->nnz > 27 * a->n_rows || a->nnz < 2 * a->n_rows || s.row_end <= s.row_begin) return false;
  if (s.q < 1 || s.q >= (int64_t{1} << 31) || s.ld % 2 || s.ld_y % 2) return false;
  const StencilPlan* sp = get_stencil_plan(const_cast<adp_csr*>(a), s.goff);
  if (!sp->valid) return false;
  const int64_t plane = sp->nx * sp->ny;
  if (s.row_begin % plane || s.row_end % plane) return false;  // whole grid planes only
  if (s.n_push) {  // boundary planes of a row partition, stored into the neighbours' halos too
    if (sp->kind == 27) {
      if (sp->classes) launch_sweep<8, 27, kShared, true>(ctx, s, *sp);
      else launch_sweep<8, 27, kExact, true>(ctx, s, *sp);
    } else {
      if (sp->classes) launch_sweep<8, 7, kUnitNeg, true>(ctx, s, *sp);
      else launch_sweep<8, 7, kExact, true>(ctx, s, *sp);
    }
  } else if (sp->kind == 27) {
    if (sp->classes) launch_sweep<8, 27, kShared>(ctx, s, *sp);
    else launch_sweep<8, 27, kExact>(ctx, s, *sp);
  } else {
    if (sp->classes) launch_sweep<8, 7, kUnitNeg>(ctx, s, *sp);
    else launch_sweep<8, 7, kExact>(ctx, s, *sp);
  }
  return true;
}

}  // namespace adp
