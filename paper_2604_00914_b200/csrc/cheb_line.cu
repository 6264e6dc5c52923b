// Fused Clenshaw step with register reuse of gathered rows along column runs
// ("line" kernel), sm_100a.
//
// Stencil-like operators (the 7- and 27-point Laplacians of configs 1, 2 and 4,
// the band of config 5) have blocks of R consecutive rows whose column patterns
// are the same pattern shifted by one per row: row r0+i holds columns
// {c + i : c in cols(r0)}. Split cols(r0) into runs of consecutive columns
// (length <= MM); for a run starting at column c0 with length m, the rows of
// the block need gathered rows c0 .. c0 + R + m - 2 -- R + m - 1 distinct rows
// instead of R * m. A warp loads them once into registers and applies them to
// all R rows; per row the products still accumulate run by run, position by
// position -- CSR (ascending column) order -- so results are bitwise the
// single-row kernels'. For config 4 (27-point, runs of 3, R = 4) this moves
// 13.5 instead of 27 gathered row panels per row through L1/L2, the resource
// the lean kernel saturates there (profiles/).
//
// Blocks whose rows do not share a shifted pattern (grid faces, tails, general
// sparsity) are processed row by row inside the same warp. The host builds the
// block -> pattern map once per operator (LinePlan) and deduplicates patterns,
// so interior blocks share one run list.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

LinePlan::~LinePlan() {
  cudaFree(d_blk_pat);
  cudaFree(d_pat_ptr);
  cudaFree(d_runs);
  cudaFree(d_prefix);
  cudaFree(d_pat_len);
}

namespace {
constexpr int64_t kMinCore = 32;  // shortest shared core worth a band block
// Longest run of consecutive columns of a row: {entry index, length}.
std::pair<int64_t, int64_t> longest_run(const int32_t* c, int64_t cnt) {
  int64_t best = 0, bl = 0, k = 0;
  while (k < cnt) {
    int64_t m = 1;
    while (k + m < cnt && c[k + m] == c[k + m - 1] + 1) ++m;
    if (m > bl) {
      bl = m;
      best = k;
    }
    k += m;
  }
  return {best, bl};
}
}  // namespace

const LinePlan* get_line_plan(adp_csr* a, int R, int mm, bool band) {
  for (auto& p : a->line_plans)
    if (p->R == R && p->mm == mm && p->band == band) return p.get();
  auto p = std::make_unique<LinePlan>();
  p->R = R;
  p->mm = mm;
  p->band = band;
  const int64_t n = a->n_rows;
  const int64_t nb = (n + R - 1) / R;
  ensure_host_copy(a);
  const std::vector<int64_t>& rp = a->h_row_ptr;
  const std::vector<int32_t>& ci = a->h_col;
  std::vector<int32_t> blk_pat(static_cast<size_t>(nb), -1);
  std::map<std::vector<int32_t>, int32_t> ids;
  std::vector<int32_t> pat_ptr{0};
  std::vector<int32_t> runs;  // {relc, k, m, 0} per run
  std::vector<int32_t> sig;
  int64_t regular = 0;
  std::vector<int32_t> prefix;  // band blocks: entries before the core, per row
  std::vector<int32_t> pat_len;
  int64_t n_band = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t r0 = b * R;
    if (r0 + R > n) break;
    const int64_t cnt = rp[r0 + 1] - rp[r0];
    if (cnt == 0 || cnt > (int64_t{1} << 20)) continue;
    bool ok = true;
    for (int i = 1; i < R && ok; ++i) {
      if (rp[r0 + i + 1] - rp[r0 + i] != cnt) {
        ok = false;
        break;
      }
      const int32_t* c0 = &ci[rp[r0]];
      const int32_t* c1 = &ci[rp[r0 + i]];
      for (int64_t k = 0; k < cnt; ++k)
        if (static_cast<int64_t>(c1[k]) != static_cast<int64_t>(c0[k]) + i) {
          ok = false;
          break;
        }
    }
    // band block: every row's longest consecutive run is row r0's shifted by i (the rest row by row)
    int64_t core_k0 = 0, core_len = cnt;
    std::vector<int32_t> pre(static_cast<size_t>(R), 0);
    bool is_band = false;
    if (!ok && band) {
      const auto [k0, len] = longest_run(&ci[rp[r0]], cnt);
      bool bok = len >= kMinCore;
      const int64_t c_start = bok ? static_cast<int64_t>(ci[rp[r0] + k0]) : 0;
      for (int i = 0; i < R && bok; ++i) {
        const int64_t ri = r0 + i, cnt_i = rp[ri + 1] - rp[ri];
        const auto [ki, li] = longest_run(&ci[rp[ri]], cnt_i);
        if (li != len || static_cast<int64_t>(ci[rp[ri] + ki]) != c_start + i || ki >= (int64_t{1} << 30)) bok = false;
        else pre[i] = static_cast<int32_t>(ki);
      }
      if (bok) {
        ok = true;
        is_band = true;
        core_k0 = k0;
        core_len = len;
      }
    }
    if (!ok) continue;
    sig.clear();
    const int32_t* c0 = &ci[rp[r0] + core_k0];
    int64_t k = 0;
    while (k < core_len) {
      int64_t m = 1;
      while (k + m < core_len && m < mm && c0[k + m] == c0[k + m - 1] + 1) ++m;
      sig.push_back(static_cast<int32_t>(static_cast<int64_t>(c0[k]) - r0));
      sig.push_back(static_cast<int32_t>(k));
      sig.push_back(static_cast<int32_t>(m));
      sig.push_back(0);
      k += m;
    }
    auto it = ids.find(sig);
    int32_t id;
    if (it == ids.end()) {
      if (ids.size() >= 65536) continue;  // too many distinct patterns: leave irregular
      id = static_cast<int32_t>(ids.size());
      ids.emplace(sig, id);
      runs.insert(runs.end(), sig.begin(), sig.end());
      pat_ptr.push_back(static_cast<int32_t>(runs.size() / 4));
      pat_len.push_back(static_cast<int32_t>(core_len));
    } else {
      id = it->second;
    }
    if (is_band) {
      if (prefix.empty()) prefix.assign(static_cast<size_t>(n), 0);
      for (int i = 0; i < R; ++i) prefix[r0 + i] = pre[i];
      ++n_band;
    }
    blk_pat[b] = id;
    ++regular;
  }
  p->n_blocks = nb;
  p->n_regular = regular;
  p->n_patterns = static_cast<int64_t>(ids.size());
  p->n_runs = static_cast<int64_t>(runs.size() / 4);
  p->regular_frac = nb > 0 ? static_cast<double>(regular) / static_cast<double>(nb) : 0.0;
  ADP_CUDA(cudaSetDevice(a->ctx->device));
  auto up = [&](void** dst, const void* src, size_t bytes) {
    ADP_CUDA(cudaMalloc(dst, std::max<size_t>(bytes, 16)));
    if (bytes) ADP_CUDA(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  };
  up(&p->d_blk_pat, blk_pat.data(), blk_pat.size() * 4);
  up(&p->d_pat_ptr, pat_ptr.data(), pat_ptr.size() * 4);
  up(&p->d_runs, runs.data(), runs.size() * 4);
  p->n_band = n_band;
  if (n_band > 0) {
    up(&p->d_prefix, prefix.data(), prefix.size() * 4);
    up(&p->d_pat_len, pat_len.data(), pat_len.size() * 4);
  }
  plan_uploads_done();
  a->line_plans.push_back(std::move(p));
  return a->line_plans.back().get();
}

namespace {

constexpr int kThreads = 256;

struct LnArgs {
  const void* row_ptr;
  const int32_t* col;
  const void* val;
  const char* g;
  const char* vin;
  const char* yin;
  char* out;
  char* wout;
  uint32_t ldg_b, ldy_b, ldo_b;
  int32_t nrows, nblk, n_panels;
  int32_t valid;  // masked launches: vectors of the single panel that exist
  int64_t goff;
  const int32_t* blk_pat;
  const int32_t* pat_ptr;
  const int4* runs;
  const int32_t* prefix;   // band plans: entries before each row's core (nullptr: no band block)
  const int32_t* pat_len;  // band plans: core entries of each pattern
  double s0, s1, s2, s3;
};

struct RealN {
  using Val = double;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double*>(p) + k); }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};
struct CplxN {
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
__device__ __forceinline__ void st_hint(void* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
template <class RP>
__device__ __forceinline__ int64_t ld_rp(const void* p, int64_t i) {
  return static_cast<int64_t>(__ldg(static_cast<const RP*>(p) + i));
}
// 2-D TMA tile load (box dims from the tensor map; rows outside the tensor read as 0)
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, int32_t x, int32_t y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma2d_hint(void* dst, const CUtensorMap* tm, int32_t x, int32_t y, uint64_t* bar,
                                           uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <class F, int CH, int R, int MM, int MODE, class RP, int MINB, int UNR, bool MASK>
__global__ void __launch_bounds__(kThreads, MINB) cheb_line_kernel(const LnArgs p) {
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  constexpr int kWarps = kThreads / 32;
  constexpr uint32_t kPB = 32 * CH * 16u;
  constexpr int kW = R + MM - 1;  // gathered rows one run needs at most
  using Val = typename F::Val;
  extern __shared__ __align__(16) uint8_t smem[];  // [8 mbarriers | pad][warp][row][V, Y]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int32_t task = static_cast<int32_t>(blockIdx.x) * kWarps + warp;
  if (task >= p.nblk * p.n_panels) return;
  const int32_t panel = task / p.nblk;
  const int32_t b = task - panel * p.nblk;
  const int32_t r0 = b * R;
  const int rows = min(R, p.nrows - r0);
  const uint32_t poff = static_cast<uint32_t>(panel) * kPB;
  const uint32_t voff = poff + lane * 16u;
  const uint64_t pol = policy_evict_first(1.0f);

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp;
  double2* my = reinterpret_cast<double2*>(smem + 128) + warp * (R * 2 * 32 * CH);
  // masked launches (ragged widths): one panel whose vectors >= p.valid do not exist
  bool ok[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) ok[c] = !MASK || c * 32 + lane < p.valid;
  const uint32_t cpb = MASK ? static_cast<uint32_t>(p.valid) * 16u : kPB;
  const int32_t pid = __ldg(p.blk_pat + b);  // operator data: before the wait
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // see pdl_wait_and_release (cheb_lean.cu)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if constexpr (kStep) {
    if (lane == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_arrive_expect_tx(bar, 2 * cpb * static_cast<uint32_t>(rows));
    }
    __syncwarp();
    if (lane < rows) {
      const uint64_t r = static_cast<uint64_t>(r0 + lane);
      bulk_g2s_hint(my + lane * (2 * 32 * CH), p.vin + r * p.ldg_b + poff, cpb, bar, pol);
      bulk_g2s_hint(my + lane * (2 * 32 * CH) + 32 * CH, p.yin + r * p.ldy_b + poff, cpb, bar, pol);
    }
  }
  const char* gb = p.g + voff;
  double2 acc[R][CH];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if constexpr (kSpmmAcc)
        acc[i][c] = (i < rows && ok[c])
                        ? *reinterpret_cast<const double2*>(p.out + static_cast<uint64_t>(r0 + i) * p.ldo_b + voff + 512 * c)
                        : make_double2(0.0, 0.0);
      else
        acc[i][c] = make_double2(0.0, 0.0);
    }
  // entries [e0, e1) of block row i, one by one (CSR order)
  auto row_entries = [&](int i, int64_t e0, int64_t e1) {
    for (int64_t e = e0; e < e1; ++e) {
      const int cidx = __ldg(p.col + e);
      const Val v = F::load(p.val, e);
      const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cidx)) * p.ldg_b);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        double2 wv = ok[c] ? __ldg(src + 32 * c) : make_double2(0.0, 0.0);
        if constexpr (kFirst) wv = scale2(p.s2, wv);
        acc[i][c] = F::mac(acc[i][c], v, wv);
      }
    }
  };
  if (pid >= 0) {  // shifted-pattern block: R full rows, or R rows sharing a shifted core (band plans)
    int64_t rs[R];
#pragma unroll
    for (int i = 0; i < R; ++i) rs[i] = ld_rp<RP>(p.row_ptr, r0 + i);
    if (p.prefix) {  // each row's entries before the core
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int32_t pre = __ldg(p.prefix + r0 + i);
        row_entries(i, rs[i], rs[i] + pre);
        rs[i] += pre;
      }
    }
    const int32_t q0 = __ldg(p.pat_ptr + pid), q1 = __ldg(p.pat_ptr + pid + 1);
#pragma unroll UNR
    for (int32_t qr = q0; qr < q1; ++qr) {
      const int4 rn = __ldg(p.runs + qr);  // {column of row r0 - r0, entry index, length, -}
      const uint32_t c0 = static_cast<uint32_t>(r0 + rn.x);
      const int m = rn.z;
      double2 w[kW][CH];
#pragma unroll
      for (int j = 0; j < kW; ++j) {
        if (j < R + m - 1) {
          const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(c0 + j) * p.ldg_b);
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            w[j][c] = ok[c] ? __ldg(src + 32 * c) : make_double2(0.0, 0.0);
            if constexpr (kFirst) w[j][c] = scale2(p.s2, w[j][c]);  // W = c_d * Y on the fly
          }
        }
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
#pragma unroll
        for (int t = 0; t < MM; ++t) {
          if (t < m) {
            const Val v = F::load(p.val, rs[i] + rn.y + t);
#pragma unroll
            for (int c = 0; c < CH; ++c) acc[i][c] = F::mac(acc[i][c], v, w[i + t][c]);
          }
        }
      }
    }
    if (p.prefix) {  // each row's entries after the core
      const int32_t clen = __ldg(p.pat_len + pid);
#pragma unroll
      for (int i = 0; i < R; ++i) row_entries(i, rs[i] + clen, ld_rp<RP>(p.row_ptr, r0 + i + 1));
    }
  } else {  // row by row, CSR order
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (i < rows) {
        const RP start = static_cast<RP>(ld_rp<RP>(p.row_ptr, r0 + i));
        const RP end = static_cast<RP>(ld_rp<RP>(p.row_ptr, r0 + i + 1));
        for (RP e = start; e < end; ++e) {
          const int cidx = __ldg(p.col + e);
          const Val v = F::load(p.val, static_cast<int64_t>(e));
          const double2* src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cidx)) * p.ldg_b);
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            double2 wv = ok[c] ? __ldg(src + 32 * c) : make_double2(0.0, 0.0);
            if constexpr (kFirst) wv = scale2(p.s2, wv);
            acc[i][c] = F::mac(acc[i][c], v, wv);
          }
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
    if (i < rows) {
      const int64_t r = r0 + i;
      const double2* own_src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(r + p.goff) * p.ldg_b);
      char* ob = p.out + static_cast<uint64_t>(r) * p.ldo_b + voff;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (!ok[c]) continue;
        double2 own = make_double2(0.0, 0.0);
        if constexpr (kNeedOwn) own = __ldg(own_src + 32 * c);
        double2 res;
        if constexpr (kStep) {
          // v = (((s0 * aw) + (s1 * w)) - v) + (s2 * y)   (cheb_filter.cpp:170-171, 176-177)
          const double2 vv = my[i * (2 * 32 * CH) + c * 32 + lane];
          const double2 yy = my[i * (2 * 32 * CH) + 32 * CH + c * 32 + lane];
          res = add2(sub2(add2(scale2(p.s0, acc[i][c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
        } else if constexpr (kFirst) {
          // w = c_d * y ; v = (2 l1) * aw + (2 l2 + c_{d-1}/c_d) * w   (cheb_filter.cpp:162-165)
          const double2 wn = scale2(p.s2, own);
          st_hint(p.wout + static_cast<uint64_t>(r) * p.ldo_b + voff + 512 * c, wn, pol);
          res = add2(scale2(p.s0, acc[i][c]), scale2(p.s1, wn));
        } else if constexpr (kDeg1) {
          // c0 * x + c1 * (l1 * ax + l2 * x)   (cheb_filter.cpp:154)
          res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[i][c]), scale2(p.s3, own))));
        } else {
          res = acc[i][c];
        }
        st_hint(ob + 512 * c, res, pol);
      }
    }
  }
}

template <class F, int CH, int R, int MM, class RP, int MINB, int UNR = 1, bool MASK = false>
bool launch_line_cfg(adp_ctx* ctx, StepMode mode, const StepArgs& s, int64_t qv, double min_regular) {
  const adp_csr* a = s.a;
  if (MASK ? (qv > 32 * CH || qv <= 32 * (CH - 1)) : qv % (32 * CH) != 0) return false;
  const LinePlan* plan = get_line_plan(const_cast<adp_csr*>(a), R, MM, true);
  if (plan->regular_frac < min_regular) return false;
  constexpr int kWarps = kThreads / 32;
  const int epv = a->dtype == ADP_C128 ? 1 : 2;
  LnArgs k{};
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
  k.nrows = static_cast<int32_t>(a->n_rows);
  k.nblk = static_cast<int32_t>(plan->n_blocks);
  k.n_panels = MASK ? 1 : static_cast<int32_t>(qv / (32 * CH));
  k.valid = static_cast<int32_t>(qv);
  k.goff = s.goff;
  k.blk_pat = static_cast<const int32_t*>(plan->d_blk_pat);
  k.pat_ptr = static_cast<const int32_t*>(plan->d_pat_ptr);
  k.runs = static_cast<const int4*>(plan->d_runs);
  k.prefix = static_cast<const int32_t*>(plan->d_prefix);
  k.pat_len = static_cast<const int32_t*>(plan->d_pat_len);
  k.s0 = s.s0;
  k.s1 = s.s1;
  k.s2 = s.s2;
  k.s3 = s.s3;
  const int64_t total = plan->n_blocks * k.n_panels;
  if (total >= (int64_t{1} << 31)) return false;
  const int grid = static_cast<int>((total + kWarps - 1) / kWarps);
  const size_t smem = mode == StepMode::Step ? 128 + static_cast<size_t>(kWarps) * R * 2 * 32 * CH * 16 : 128;
  auto run = [&](auto kern) {
    if (smem > 48 * 1024)
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    launch_pdl(ctx, kern, dim3(grid), dim3(kThreads), smem, k);
  };
  switch (mode) {
    case StepMode::First: run(cheb_line_kernel<F, CH, R, MM, 0, RP, MINB, UNR, MASK>); break;
    case StepMode::Step: run(cheb_line_kernel<F, CH, R, MM, 1, RP, MINB, UNR, MASK>); break;
    case StepMode::Deg1: run(cheb_line_kernel<F, CH, R, MM, 2, RP, MINB, UNR, MASK>); break;
    case StepMode::Spmm: run(cheb_line_kernel<F, CH, R, MM, 3, RP, MINB, UNR, MASK>); break;
    case StepMode::SpmmAcc: run(cheb_line_kernel<F, CH, R, MM, 4, RP, MINB, UNR, MASK>); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
  return true;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

// Row-major fp64 matrix (rows x width words, row pitch ld_b bytes) tiled in
// boxes of box_rows x box_words.
CUtensorMap make_map(const void* base, int64_t rows, int64_t width, int64_t ld_b, int box_rows, int box_words) {
  auto enc = tensor_map_encoder();
  if (!enc) fail(ADP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(width), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_b)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_words), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ADP_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

template <class F, class RP>
bool dispatch_line(adp_ctx* ctx, StepMode mode, const StepArgs& s, int64_t qv) {
  // variant 3: the line kernel forced (its automatic geometry: R = 2 rows, runs <= 3, 1 KB panels)
  return ctx->variant == 3 && launch_line_cfg<F, 2, 2, 3, RP, 3>(ctx, mode, s, qv, 0.0);
}

}  // namespace

CUtensorMap make_tensor_map_f64(const void* base, int64_t rows, int64_t width, int64_t ld_b, int box_rows,
                                int box_words) {
  return make_map(base, rows, width, ld_b, box_rows, box_words);
}

// Automatic choice (variant 0): the line kernel where it measured faster than
// the lean kernel (tools/tune_step.py, profiles/r01_kernel_evolution.md): long
// stencil rows (config 4: 27 entries, gather-latency bound) whose row blocks are
// mostly shifted copies of one pattern. Short-row operators (configs 1-3, the
// config-1 solve) stay on the lean kernel, which is faster there. A ragged
// width runs as full 64-vector panels plus one masked launch for the rest.
template <class F, class RP>
bool auto_line(adp_ctx* ctx, StepMode mode, const StepArgs& s, int64_t qv) {
  const adp_csr* a = s.a;
  const bool long_rows = a->nnz >= 12 * a->n_rows;
  if (!long_rows || a->dtype != ADP_F64 || ctx->panel_cols != 0) return false;
  // the cube kernel where the operator has 3-D shifted blocks: every panel in one launch when the last
  // panel is at least half full (masked), else its full panels and the line kernel's masked tail;
  // without 3-D blocks the line kernel's full panels plus one masked launch for the rest
  const int64_t full = qv / 64 * 64, rem = qv - full;
  if (qv >= 64 && (rem == 0 || rem >= 32) && launch_cube_auto(ctx, mode, s, qv)) return true;
  if (full > 0) {
    StepArgs t = s;
    t.q = full * 2;
    if (!launch_cube_auto(ctx, mode, t, full) && !launch_line_cfg<F, 2, 2, 3, RP, 3>(ctx, mode, t, full, 0.5))
      return false;
  } else if (get_line_plan(const_cast<adp_csr*>(a), 2, 3)->regular_frac < 0.5) {
    return false;
  }
  if (rem > 0) {  // column-offset pointers, like the lean kernel's ragged split
    StepArgs t = s;
    const int64_t off = full * 16;
    auto shift = [&](const void* ptr) -> void* {
      return ptr ? const_cast<char*>(static_cast<const char*>(ptr) + off) : nullptr;
    };
    t.gsrc = shift(s.gsrc);
    t.vin = shift(s.vin);
    t.yin = shift(s.yin);
    t.out = shift(s.out);
    t.wout = shift(s.wout);
    t.q = rem * 2;
    const bool ok = rem <= 32 ? launch_line_cfg<F, 1, 2, 3, RP, 4, 1, true>(ctx, mode, t, rem, 0.0)
                              : launch_line_cfg<F, 2, 2, 3, RP, 3, 1, true>(ctx, mode, t, rem, 0.0);
    if (!ok) fail(ADP_ERR_RUNTIME, "line kernel: ragged tail launch failed");
  }
  return true;
}

bool launch_step_line(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  const adp_csr* a = s.a;
  if (a->n_rows >= (int64_t{1} << 30)) return false;
  const bool cplx = a->dtype == ADP_C128;
  const int epv = cplx ? 1 : 2;
  const int64_t qv = (s.q + epv - 1) / epv;  // odd real widths: the padding column of the (even) ld rides along
  for (int64_t ld : {s.ld, s.ld_y, s.ld_out})
    if (ld % epv != 0 || (ld / epv) * 16 >= (int64_t{1} << 32)) return false;
  if (s.row_begin != 0 || s.row_end != a->n_rows) {
    // a row range (a rank's interior rows in the row-partitioned filter): the cube kernel plans its
    // blocks inside the range; the line kernel and ragged tails need whole operators
    return ctx->variant == 0 && !cplx && ctx->auto_line && a->nnz >= 12 * a->n_rows && ctx->panel_cols == 0 &&
           qv >= 64 && launch_cube_auto(ctx, mode, s, qv);
  }
  if (ctx->variant == 0) {
    if (cplx || !ctx->auto_line) return false;
    return a->rp64 ? auto_line<RealN, int64_t>(ctx, mode, s, qv) : auto_line<RealN, int32_t>(ctx, mode, s, qv);
  }
  if (cplx) return a->rp64 ? dispatch_line<CplxN, int64_t>(ctx, mode, s, qv) : dispatch_line<CplxN, int32_t>(ctx, mode, s, qv);
  return a->rp64 ? dispatch_line<RealN, int64_t>(ctx, mode, s, qv) : dispatch_line<RealN, int32_t>(ctx, mode, s, qv);
}

}  // namespace adp
