// Fused Clenshaw step with register reuse of gathered rows across a 2-D/3-D
// block of rows ("cube" kernel), sm_100a.
//
// The line kernel (cheb_line.cu) reuses gathered W rows along one run of
// consecutive columns shared by R consecutive rows. On a 3-D stencil the rows
// of neighbouring grid lines share whole runs too: row r + sy (next y line)
// reads the x-run at column c + sy, which row r reads as its own y+1 run. A
// block here is L lines of R consecutive rows, line l starting at r0 + off[l]
// (off = {j*sy + k*sz}); when every row of the block holds the pattern of r0
// shifted by its offset, the block's distinct runs ("items") are the union of
// the lines' runs, each loaded ONCE (R + m - 1 rows into registers) and applied
// to every line that uses it. Items are visited in ascending column order and a
// line's runs are a subsequence of them, so every row still accumulates its
// products in ascending column order -- CSR order, the reference's maspmm order
// (tiled_matrix.hpp:200-205) -- and the result is bitwise the lean kernel's.
// Config 4 (27-point stencil, 2 x 2 lines of 2 rows): 16 items of 4 rows for 8
// output rows, 8 gathered row panels per row instead of 27 (lean) or 18 (line).
//
// Blocks whose rows do not share the shifted pattern (grid faces) run row by
// row inside the warp; rows that cannot be grouped into a full block (grid
// dimensions not divisible by the block) form remainder blocks of listed rows.
// The host derives sy / sz from the operator's dominant pattern (the shifts
// under which most of its runs coincide), once per operator (CubePlan).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <cstdint>
#include <map>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

CUtensorMap make_tensor_map_f64(const void* base, int64_t rows, int64_t width, int64_t ld_b, int box_rows,
                                int box_words);  // cheb_line.cu

CubePlan::~CubePlan() {
  cudaFree(d_blk);
  cudaFree(d_pat_ptr);
  cudaFree(d_items);
  cudaFree(d_rem);
  cudaFree(d_pat_nv);
  cudaFree(d_vals);
}

namespace {

// runs of consecutive columns (length <= mm) of a relative pattern: {start, entry index, length}
void split_runs(const int64_t* rel, int64_t cnt, int mm, std::vector<std::array<int64_t, 3>>& out) {
  out.clear();
  int64_t k = 0;
  while (k < cnt) {
    int64_t m = 1;
    while (k + m < cnt && m < mm && rel[k + m] == rel[k + m - 1] + 1) ++m;
    out.push_back({rel[k], k, m});
    k += m;
  }
}

// The shifts (sy, sz) under which the dominant row pattern's runs coincide most.
bool detect_strides(const adp_csr* a, int mm, int64_t& sy, int64_t& sz) {
  const std::vector<int64_t>& rp = a->h_row_ptr;
  const std::vector<int32_t>& ci = a->h_col;
  const int64_t n = a->n_rows;
  std::map<std::vector<int64_t>, int64_t> freq;
  const int64_t step = std::max<int64_t>(1, n / 4096);
  std::vector<int64_t> rel;
  for (int64_t r = step / 2; r < n; r += step) {
    const int64_t cnt = rp[r + 1] - rp[r];
    if (cnt <= 0 || cnt > 4096) continue;
    rel.resize(static_cast<size_t>(cnt));
    for (int64_t k = 0; k < cnt; ++k) rel[k] = static_cast<int64_t>(ci[rp[r] + k]) - r;
    ++freq[rel];
  }
  if (freq.empty()) return false;
  auto best = std::max_element(freq.begin(), freq.end(), [](auto& x, auto& y) { return x.second < y.second; });
  std::vector<std::array<int64_t, 3>> runs;
  split_runs(best->first.data(), static_cast<int64_t>(best->first.size()), mm, runs);
  std::vector<int64_t> starts;
  for (auto& rn : runs) starts.push_back(rn[0]);
  std::map<int64_t, int> ov;
  for (int64_t si : starts)
    for (int64_t sj : starts)
      if (sj > si) ov[sj - si] += 1;
  int maxov = 0;
  for (auto& [d, c] : ov) maxov = std::max(maxov, c);
  if (maxov < 2) return false;
  sy = 0;
  sz = 0;
  for (auto& [d, c] : ov) {  // ascending d
    if (c != maxov) continue;
    if (sy == 0) {
      sy = d;
    } else if (sz == 0 && !(d % sy == 0 && d / sy <= 4)) {
      sz = d;
    }
  }
  return sy > 0;
}

}  // namespace

// Blocks cover rows [rb, re) (a launch's row range: the whole operator, or a rank's interior rows in
// the row-partitioned filter); rows of the range outside every full block are listed as remainder.
const CubePlan* get_cube_plan(adp_csr* a, int R, int ly, int lz, int mm, int64_t rb, int64_t re) {
  for (auto& p : a->cube_plans)
    if (p->R == R && p->ly == ly && p->lz == lz && p->mm == mm && p->row_begin == rb && p->row_end == re)
      return p.get();
  auto p = std::make_unique<CubePlan>();
  p->R = R;
  p->ly = ly;
  p->lz = lz;
  p->mm = mm;
  p->row_begin = rb;
  p->row_end = re;
  const int L = ly * lz;
  ensure_host_copy(a);
  int64_t sy = 0, sz = 0;
  const bool have = detect_strides(a, mm, sy, sz) && (ly == 1 || sy > 0) && (lz == 1 || sz > 0);
  p->sy = sy;
  p->sz = sz;
  const int64_t n = a->n_rows;
  if (!have || L > 8 || n >= (int64_t{1} << 30)) {
    a->cube_plans.push_back(std::move(p));
    return a->cube_plans.back().get();
  }
  for (int k = 0; k < lz; ++k)
    for (int j = 0; j < ly; ++j) p->off[k * ly + j] = static_cast<int32_t>(j * sy + k * sz);
  const std::vector<int64_t>& rp = a->h_row_ptr;
  const std::vector<int32_t>& ci = a->h_col;
  std::vector<uint8_t> taken(static_cast<size_t>(re - rb), 0);  // indexed r - rb
  std::vector<int32_t> blk;  // {r0, pattern} pairs
  std::vector<int32_t> rem;
  std::map<std::vector<int32_t>, int32_t> ids;
  std::vector<int32_t> pat_ptr{0};
  std::vector<int32_t> items;  // 4 int32 per item: {start - r0, length, line mask, 0}
  std::vector<int32_t> pat_nv;  // values per block of each pattern
  const size_t vb = a->dtype == ADP_C128 ? 16 : 8;
  const int cs = (R * mm + 1) / 2 * 2;  // values per (item, line) chunk: [i * mm + t], padded even
  const auto* hv = static_cast<const uint8_t*>(a->h_values);
  std::vector<uint8_t> vals;  // per regular block: its chunks in item order
  std::vector<int64_t> rel;
  std::vector<std::array<int64_t, 3>> runs;
  std::map<std::pair<int64_t, int64_t>, std::array<int32_t, 8>> union_items;
  std::vector<int32_t> sig;
  int64_t regular = 0;
  for (int64_t r0 = rb; r0 < re; ++r0) {
    if (taken[r0 - rb]) continue;
    bool fits = true;
    for (int l = 0; l < L && fits; ++l)
      for (int i = 0; i < R && fits; ++i) {
        const int64_t r = r0 + p->off[l] + i;
        if (r >= re || taken[r - rb]) fits = false;
      }
    if (!fits) {
      taken[r0 - rb] = 1;
      rem.push_back(static_cast<int32_t>(r0));
      continue;
    }
    for (int l = 0; l < L; ++l)
      for (int i = 0; i < R; ++i) taken[r0 + p->off[l] + i - rb] = 1;
    int32_t pid = -1;
    const int64_t cnt = rp[r0 + 1] - rp[r0];
    bool ok = cnt > 0 && cnt < 32768;
    for (int l = 0; l < L && ok; ++l)
      for (int i = 0; i < R && ok; ++i) {
        const int64_t d = p->off[l] + i, r = r0 + d;
        if (rp[r + 1] - rp[r] != cnt) {
          ok = false;
          break;
        }
        for (int64_t k = 0; k < cnt; ++k)
          if (static_cast<int64_t>(ci[rp[r] + k]) != static_cast<int64_t>(ci[rp[r0] + k]) + d) {
            ok = false;
            break;
          }
      }
    if (ok) {
      rel.resize(static_cast<size_t>(cnt));
      for (int64_t k = 0; k < cnt; ++k) rel[k] = static_cast<int64_t>(ci[rp[r0] + k]) - r0;
      split_runs(rel.data(), cnt, mm, runs);
      union_items.clear();
      for (int l = 0; l < L; ++l)
        for (auto& rn : runs) {
          auto& it = union_items[{rn[0] + p->off[l], rn[2]}];  // key (start, length): ascending start
          it[2] |= 1 << l;
          const int32_t kk = static_cast<int32_t>(rn[1]);
          it[4 + l / 2] |= kk << (16 * (l % 2));
        }
      sig.clear();
      int64_t nv = 0;
      for (auto& [key, it] : union_items) {
        sig.push_back(static_cast<int32_t>(key.first));
        sig.push_back(static_cast<int32_t>(key.second));
        sig.push_back(it[2]);
        sig.push_back(0);
        nv += static_cast<int64_t>(__builtin_popcount(static_cast<uint32_t>(it[2]))) * cs;
      }
      if (nv * static_cast<int64_t>(vb) <= kCubeValueSlot * static_cast<int64_t>(vb / 8)) {
        auto f = ids.find(sig);
        if (f != ids.end()) {
          pid = f->second;
        } else if (ids.size() < 65536) {
          pid = static_cast<int32_t>(ids.size());
          ids.emplace(sig, pid);
          items.insert(items.end(), sig.begin(), sig.end());
          pat_ptr.push_back(static_cast<int32_t>(items.size() / 4));
          pat_nv.push_back(static_cast<int32_t>(nv));
        }
      }
      if (pid >= 0) {  // the block's values in the order the kernel consumes them
        const size_t v0 = vals.size();
        vals.resize(v0 + static_cast<size_t>(nv) * vb, 0);
        uint8_t* dst = vals.data() + v0;
        for (auto& [key, it] : union_items)
          for (int l = 0; l < L; ++l) {
            if (!(it[2] & (1 << l))) continue;
            const int64_t kk = (it[4 + l / 2] >> (16 * (l % 2))) & 0xffff;
            for (int i = 0; i < R; ++i)
              for (int64_t t = 0; t < key.second; ++t)
                std::memcpy(dst + (i * mm + t) * vb, hv + (rp[r0 + p->off[l] + i] + kk + t) * vb, vb);
            dst += cs * vb;
          }
        blk.push_back(static_cast<int32_t>(r0));
        blk.push_back(pid);
        const int64_t vi = static_cast<int64_t>(v0 / vb);
        blk.push_back(static_cast<int32_t>(vi & 0xffffffff));
        blk.push_back(static_cast<int32_t>(vi >> 32));
        ++regular;
        continue;
      }
    }
    blk.push_back(static_cast<int32_t>(r0));
    blk.push_back(-1);
    blk.push_back(0);
    blk.push_back(0);
  }
  // remainder rows: blocks of up to L * R listed rows (pattern -2, r0 = index into the list)
  const int32_t per = L * R;
  for (size_t i = 0; i < rem.size(); i += per) {
    blk.push_back(static_cast<int32_t>(i));
    blk.push_back(-2);
    blk.push_back(0);
    blk.push_back(0);
  }
  p->n_blocks = static_cast<int64_t>(blk.size() / 4);
  p->n_regular = regular;
  p->n_rem = static_cast<int64_t>(rem.size());
  p->n_patterns = static_cast<int64_t>(ids.size());
  p->n_items = static_cast<int64_t>(items.size() / 4);
  p->regular_rows_frac = re > rb ? static_cast<double>(regular * per) / static_cast<double>(re - rb) : 0.0;
  ADP_CUDA(cudaSetDevice(a->ctx->device));
  auto up = [&](void** dst, const void* src, size_t bytes) {
    ADP_CUDA(cudaMalloc(dst, std::max<size_t>(bytes, 16)));
    if (bytes) ADP_CUDA(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  };
  up(&p->d_blk, blk.data(), blk.size() * 4);
  up(&p->d_pat_ptr, pat_ptr.data(), pat_ptr.size() * 4);
  up(&p->d_items, items.data(), items.size() * 4);
  up(&p->d_rem, rem.data(), rem.size() * 4);
  up(&p->d_pat_nv, pat_nv.data(), pat_nv.size() * 4);
  up(&p->d_vals, vals.data(), vals.size());
  p->valid = true;
  plan_uploads_done();
  a->cube_plans.push_back(std::move(p));
  return a->cube_plans.back().get();
}

namespace {


struct CbArgs {
  const void* row_ptr;
  const int32_t* col;
  const void* val;
  const char* g;
  const char* vin;
  const char* yin;
  char* out;
  char* wout;
  uint32_t ldg_b, ldy_b, ldo_b;
  int32_t nblk, n_panels, n_groups, gp;  // gp: panels per task
  int32_t nrem;
  int32_t valid_vec;  // 16-byte vectors of a row that exist (the last panel may be partial)
  int64_t goff;
  const int4* blk;
  const int32_t* pat_ptr;
  const int32_t* pat_nv;
  const int4* items;
  const int32_t* rem;
  const void* vals;
  int32_t off[8];
  double s0, s1, s2, s3;
};

struct RealC {
  using Val = double;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double*>(p) + k); }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, w.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, w.y));
    return acc;
  }
};
struct CplxC {
  using Val = double2;
  static __device__ __forceinline__ Val load(const void* p, int64_t k) { return __ldg(static_cast<const double2*>(p) + k); }
  static __device__ __forceinline__ double2 mac(double2 acc, Val v, double2 w) {
    // the complex accumulation of every kernel (cheb_line.cu CplxN, oracle.cpp cplx mac)
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
__device__ __forceinline__ void st_hint(void* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
template <class RP>
__device__ __forceinline__ int64_t ld_rp(const void* p, int64_t i) {
  return static_cast<int64_t>(__ldg(static_cast<const RP*>(p) + i));
}

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <class F>
__host__ __device__ constexpr uint32_t cube_value_slot() {
  return static_cast<uint32_t>(kCubeValueSlot) * (sizeof(typename F::Val) / 8);
}
// rows per ring stage: one item's R + MM - 1 gathered rows, or (Step) a line's V and Y rows. (The own W
// rows through the ring too -- 3R rows per stage -- measured slower: the larger stages cost occupancy.)
template <int R, int MM, int MODE>
__host__ __device__ constexpr int cube_stage_rows() {
  return MODE == static_cast<int>(StepMode::Step) && 2 * R > R + MM - 1 ? 2 * R : R + MM - 1;
}
template <class F, int CH, int R, int MM, int S, int MODE>
__host__ __device__ constexpr uint32_t cube_warp_smem() {
  return cube_value_slot<F>() + static_cast<uint32_t>(S) * cube_stage_rows<R, MM, MODE>() * 32 * CH * 16;
}
// 2-D TMA tile load (box from the tensor map; rows past the end read as 0)
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

// One warp (SP = 1) or a pair of warps (SP = 2) per task (block, group of panels). The
// task's stream of TMA tile copies -- per panel, each item's R + m - 1 gathered rows, then
// (Step mode) each line's V and Y rows -- runs through a ring of S shared-memory stages,
// S entries ahead of the consumers and across panel boundaries, so the gathers' and
// streams' latency is covered by copies in flight rather than by registers. The block's
// values sit in shared memory for the whole task in the order the items consume them.
// With SP = 2 both warps read every item from the shared ring and each accumulates half
// of the block's lines (half the registers, half the shared memory per warp: more
// resident warps); they meet at a pair barrier before a stage is refilled. Remainder
// blocks (listed rows) read V / Y directly.
template <class F, int CH, int R, int L, int MM, int S, int MODE, class RP, int MINB, int SP, bool LAZY, int NT>
__global__ void __launch_bounds__(NT, MINB)
    cheb_cube_kernel(const CbArgs p, const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_v,
                     const __grid_constant__ CUtensorMap tm_y) {
  static_assert(SP == 1 || SP == 2, "one warp or a warp pair per task");
  static_assert(L % SP == 0, "lines split evenly over the warps of a task");
  constexpr bool kStep = MODE == static_cast<int>(StepMode::Step);
  constexpr bool kFirst = MODE == static_cast<int>(StepMode::First);
  constexpr bool kDeg1 = MODE == static_cast<int>(StepMode::Deg1);
  constexpr bool kSpmmAcc = MODE == static_cast<int>(StepMode::SpmmAcc);
  constexpr bool kNeedOwn = kStep || kFirst || kDeg1;
  constexpr int kTasks = NT / 32 / SP;  // tasks per CTA
  constexpr int LW = L / SP;                  // lines per warp
  constexpr uint32_t kPB = 32 * CH * 16u;
  constexpr int32_t kPE = static_cast<int32_t>(kPB / 8);  // panel width in fp64 words
  constexpr int kW = R + MM - 1;
  constexpr int kSR = cube_stage_rows<R, MM, MODE>();
  constexpr int kCS = (R * MM + 1) / 2 * 2;  // values per (item, line) chunk: [i * MM + t]
  using Val = typename F::Val;
  constexpr uint32_t kVS = cube_value_slot<F>();
  constexpr uint32_t kWB = cube_warp_smem<F, CH, R, MM, S, MODE>();  // per task
  // [(S + 1) mbarriers per task, 128 B aligned][task: block values | S stages of kSR row panels]
  constexpr uint32_t kBarB = ((kTasks * (S + 1) * 8) + 127) / 128 * 128;
  extern __shared__ __align__(128) uint8_t smem[];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int slot = warp / SP, half = warp % SP;
  const int32_t task = static_cast<int32_t>(blockIdx.x) * kTasks + slot;
  if (task >= p.nblk * p.n_groups) return;  // both warps of a pair leave together
  const int32_t grp = task / p.nblk;
  const int32_t b = task - grp * p.nblk;
  const int4 bk = __ldg(p.blk + b);  // {r0 (or index into the remainder list), pattern id, value offset}
  const int32_t r0 = bk.x, pid = bk.y;
  const int32_t pan0 = grp * p.gp, pan1 = min(pan0 + p.gp, p.n_panels);
  const uint64_t pol = policy_evict_first();
  uint64_t* bar_v = reinterpret_cast<uint64_t*>(smem) + (S + 1) * slot;
  uint64_t* bar_r = bar_v + 1;  // one per ring stage
  uint8_t* ws = smem + kBarB + slot * kWB;
  const Val* sv = reinterpret_cast<const Val*>(ws);
  double2* ring = reinterpret_cast<double2*>(ws + kVS);
  const bool producer = half == 0;
  auto task_sync = [&]() {
    if constexpr (SP == 1) {
      __syncwarp();
    } else {
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + slot), "r"(32 * SP) : "memory");
    }
  };

  // line lw of this warp is block line half * LW + lw; its row i -> r0 + off[l] + i (remainder: listed)
  auto row_of = [&](int l, int i, bool& ok) -> int32_t {
    if (pid == -2) {
      const int32_t idx = r0 + l * R + i;
      ok = idx < p.nrem;
      return ok ? __ldg(p.rem + idx) : 0;
    }
    ok = true;
    return r0 + p.off[l] + i;
  };
  int32_t q0 = 0, nit = 0;
  if (producer && lane == 0) {
    for (int st = 0; st <= S; ++st) mbar_init(bar_v + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (pid >= 0) {
    q0 = __ldg(p.pat_ptr + pid);
    nit = __ldg(p.pat_ptr + pid + 1) - q0;
    if (producer && lane == 0) {  // the block's values, in consumption order, once per task
      const uint32_t bytes = static_cast<uint32_t>(__ldg(p.pat_nv + pid)) * static_cast<uint32_t>(sizeof(Val));
      const int64_t vo = (static_cast<int64_t>(static_cast<uint32_t>(bk.w)) << 32) | static_cast<uint32_t>(bk.z);
      mbar_arrive_expect_tx(bar_v, bytes);
      bulk_g2s(ws, static_cast<const Val*>(p.vals) + vo, bytes, bar_v);
    }
  }
  task_sync();  // barriers initialised before any warp of the task waits on them
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // see pdl_wait_and_release (cheb_lean.cu)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const bool vy = kStep && pid != -2;  // V / Y rows through the ring
  const int32_t per = nit + (vy ? L : 0);
  const int32_t nstream = per * (pan1 - pan0);
  // producer state (warp-uniform): next stream entry (panel pk, entry e) and its stage.
  // V / Y entries are interleaved over the warps: entry nit + e carries line (e % SP) * LW + e / SP.
  int32_t pe = 0, ppk = 0, pst = 0;
  const int32_t npan = nstream > 0 ? pan1 - pan0 : 0;
  auto produce = [&]() {  // the producer warp's lane 0 issues the copies of the next stream entry
    if (!producer || ppk >= npan) return;
    if (lane == 0) {
      double2* dst = ring + pst * kSR * 32 * CH;
      const int32_t x = (pan0 + ppk) * kPE;
      if (pe < nit) {
        const int4 h = __ldg(p.items + q0 + pe);
        mbar_arrive_expect_tx(bar_r + pst, kW * kPB);
        tma2d(dst, &tm_w, x, r0 + h.x, bar_r + pst);
      } else {
        const int32_t e = pe - nit;
        const int32_t row0 = r0 + p.off[(e % SP) * LW + e / SP];
        mbar_arrive_expect_tx(bar_r + pst, 2 * R * kPB);
        tma2d_hint(dst, &tm_v, x, row0, bar_r + pst, pol);
        tma2d_hint(dst + R * 32 * CH, &tm_y, x, row0, bar_r + pst, pol);
      }
    }
    pst = pst + 1 == S ? 0 : pst + 1;
    if (++pe == per) {
      pe = 0;
      ++ppk;
    }
  };
#pragma unroll
  for (int k = 0; k < S; ++k) produce();
  if (pid >= 0) mbar_wait(bar_v, 0);
  int32_t cst = 0;   // consumer stage
  uint32_t cph = 0;  // its phase parity
  auto consumed = [&]() {  // every warp of the task has read the stage: refill it
    task_sync();
    produce();
    if (++cst == S) {
      cst = 0;
      cph ^= 1u;
    }
  };

  for (int32_t panel = pan0; panel < pan1; ++panel) {
    const uint32_t voff = static_cast<uint32_t>(panel) * kPB + lane * 16u;
    const char* gb = p.g + voff;
    bool okc[CH];  // lanes past a ragged width: their tiles read zeros (TMA), they load and store nothing
#pragma unroll
    for (int c = 0; c < CH; ++c) okc[c] = static_cast<int32_t>(panel * 32 * CH + c * 32 + lane) < p.valid_vec;
    double2 acc[LW][R][CH];
#pragma unroll
    for (int lw = 0; lw < LW; ++lw)
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          if constexpr (kSpmmAcc) {
            bool ok;
            const int32_t r = row_of(half * LW + lw, i, ok);
            acc[lw][i][c] = ok && okc[c]
                                ? *reinterpret_cast<const double2*>(p.out + static_cast<uint64_t>(r) * p.ldo_b + voff + 512 * c)
                                : make_double2(0.0, 0.0);
          } else {
            acc[lw][i][c] = make_double2(0.0, 0.0);
          }
        }
    if (pid >= 0) {  // shifted-pattern block: the union of the lines' runs, ascending
      int32_t vo = 0;  // chunk offset of the item's first active line in the block's values
      for (int32_t qi = 0; qi < nit; ++qi) {
        const int4 h = __ldg(p.items + q0 + qi);  // {start - r0, length, line mask, -}
        const int m = h.y;
        const uint32_t mask = static_cast<uint32_t>(h.z);
        mbar_wait(bar_r + cst, cph);
        const double2* sr = ring + cst * kSR * 32 * CH + lane;
        double2 w[LAZY ? 1 : kW][CH];
        if constexpr (!LAZY) {  // the item's rows into registers, the stage released at once
#pragma unroll
          for (int j = 0; j < kW; ++j)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              w[j][c] = sr[(j * CH + c) * 32];
              if constexpr (kFirst) w[j][c] = scale2(p.s2, w[j][c]);  // W = c_d * Y on the fly
            }
          consumed();
        }
#pragma unroll
        for (int lw = 0; lw < LW; ++lw) {
          const int l = half * LW + lw;
          if (mask & (1u << l)) {
            // chunks are stored per item in ascending line order
            const int32_t co = vo + kCS * __popc(mask & ((1u << l) - 1u));
            Val v[kCS];
            if constexpr (sizeof(Val) == 8) {
              const double2* cv = reinterpret_cast<const double2*>(sv + co);
#pragma unroll
              for (int e = 0; e < kCS / 2; ++e) {
                const double2 t2 = cv[e];
                v[2 * e] = t2.x;
                v[2 * e + 1] = t2.y;
              }
            } else {
#pragma unroll
              for (int e = 0; e < kCS; ++e) v[e] = sv[co + e];
            }
            if constexpr (LAZY) {
              // one gathered row at a time, read from the stage: row j feeds (i, t = j - i); for a
              // fixed row i, t ascends with j, so each row still accumulates in column order
#pragma unroll
              for (int j = 0; j < kW; ++j) {
                if (j < R + m - 1) {
#pragma unroll
                  for (int c = 0; c < CH; ++c) {
                    w[0][c] = sr[(j * CH + c) * 32];
                    if constexpr (kFirst) w[0][c] = scale2(p.s2, w[0][c]);
                  }
#pragma unroll
                  for (int i = 0; i < R; ++i) {
                    const int t = j - i;
                    if (t >= 0 && t < MM && t < m) {
#pragma unroll
                      for (int c = 0; c < CH; ++c) acc[lw][i][c] = F::mac(acc[lw][i][c], v[i * MM + t], w[0][c]);
                    }
                  }
                }
              }
            } else if (m == MM) {  // position-major: the R x CH accumulators' chains interleave
#pragma unroll
              for (int t = 0; t < MM; ++t)
#pragma unroll
                for (int i = 0; i < R; ++i)
#pragma unroll
                  for (int c = 0; c < CH; ++c) acc[lw][i][c] = F::mac(acc[lw][i][c], v[i * MM + t], w[i + t][c]);
            } else {
#pragma unroll
              for (int i = 0; i < R; ++i)
#pragma unroll
                for (int t = 0; t < MM; ++t)
                  if (t < m) {
#pragma unroll
                    for (int c = 0; c < CH; ++c) acc[lw][i][c] = F::mac(acc[lw][i][c], v[i * MM + t], w[i + t][c]);
                  }
            }
          }
        }
        if constexpr (LAZY) consumed();  // every read of the stage done
        vo += kCS * __popc(mask);
      }
    } else {  // row by row, CSR order
#pragma unroll
      for (int lw = 0; lw < LW; ++lw)
#pragma unroll
        for (int i = 0; i < R; ++i) {
          bool ok;
          const int32_t r = row_of(half * LW + lw, i, ok);
          if (ok) {
            const RP start = static_cast<RP>(ld_rp<RP>(p.row_ptr, r));
            const RP end = static_cast<RP>(ld_rp<RP>(p.row_ptr, r + 1));
            for (RP e = start; e < end; ++e) {
              const int cidx = __ldg(p.col + e);
              const Val v = F::load(p.val, static_cast<int64_t>(e));
              const double2* src =
                  reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(static_cast<uint32_t>(cidx)) * p.ldg_b);
#pragma unroll
              for (int c = 0; c < CH; ++c) {
                double2 wv = okc[c] ? __ldg(src + 32 * c) : make_double2(0.0, 0.0);
                if constexpr (kFirst) wv = scale2(p.s2, wv);
                acc[lw][i][c] = F::mac(acc[lw][i][c], v, wv);
              }
            }
          }
        }
    }
    // epilogue: V / Y entries arrive interleaved over the warps (lw, then the warp that owns it)
#pragma unroll
    for (int lw = 0; lw < LW; ++lw) {
#pragma unroll
      for (int hh = 0; hh < SP; ++hh) {
        const double2* sr = ring + cst * kSR * 32 * CH + lane;  // line hh * LW + lw's V / Y rows (Step, vy)
        if constexpr (kStep) {
          if (vy) mbar_wait(bar_r + cst, cph);
        }
        if (hh == half) {
          const int l = half * LW + lw;
#pragma unroll
          for (int i = 0; i < R; ++i) {
            bool ok;
            const int64_t r = row_of(l, i, ok);
            if (!ok) continue;
            const double2* own_src = reinterpret_cast<const double2*>(gb + static_cast<uint64_t>(r + p.goff) * p.ldg_b);
            char* ob = p.out + static_cast<uint64_t>(r) * p.ldo_b + voff;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              if (!okc[c]) continue;
              double2 own = make_double2(0.0, 0.0);
              if constexpr (kNeedOwn) own = __ldg(own_src + 32 * c);
              double2 res;
              if constexpr (kStep) {
                // v = (((s0 * aw) + (s1 * w)) - v) + (s2 * y)   (cheb_filter.cpp:170-171, 176-177)
                double2 vv, yy;
                if (vy) {
                  vv = sr[(i * CH + c) * 32];
                  yy = sr[((R + i) * CH + c) * 32];
                } else {
                  vv = __ldg(reinterpret_cast<const double2*>(p.vin + static_cast<uint64_t>(r) * p.ldg_b + voff + 512 * c));
                  yy = __ldg(reinterpret_cast<const double2*>(p.yin + static_cast<uint64_t>(r) * p.ldy_b + voff + 512 * c));
                }
                res = add2(sub2(add2(scale2(p.s0, acc[lw][i][c]), scale2(p.s1, own)), vv), scale2(p.s2, yy));
              } else if constexpr (kFirst) {
                // w = c_d * y ; v = (2 l1) * aw + (2 l2 + c_{d-1}/c_d) * w   (cheb_filter.cpp:162-165)
                const double2 wn = scale2(p.s2, own);
                st_hint(p.wout + static_cast<uint64_t>(r) * p.ldo_b + voff + 512 * c, wn, pol);
                res = add2(scale2(p.s0, acc[lw][i][c]), scale2(p.s1, wn));
              } else if constexpr (kDeg1) {
                // c0 * x + c1 * (l1 * ax + l2 * x)   (cheb_filter.cpp:154)
                res = add2(scale2(p.s0, own), scale2(p.s1, add2(scale2(p.s2, acc[lw][i][c]), scale2(p.s3, own))));
              } else {
                res = acc[lw][i][c];
              }
              st_hint(ob + 512 * c, res, pol);
            }
          }
        }
        if constexpr (kStep) {
          if (vy) consumed();
        }
      }
    }
  }
}

template <class F, int CH, int R, int LY, int LZ, int MM, int S, class RP, int MINB, int SP = 1, bool LAZY = false,
          int NT = 256>
bool launch_cube_cfg(adp_ctx* ctx, StepMode mode, const StepArgs& s, int64_t qv, int gp, double min_regular) {
  constexpr int L = LY * LZ;
  const adp_csr* a = s.a;
  if (qv < 32 * CH) return false;  // a ragged last panel runs masked; narrower blocks take other kernels
  const CubePlan* plan = get_cube_plan(const_cast<adp_csr*>(a), R, LY, LZ, MM, s.row_begin, s.row_end);
  if (!plan->valid || plan->regular_rows_frac < min_regular) return false;
  constexpr int kWarps = NT / 32;
  const int epv = a->dtype == ADP_C128 ? 1 : 2;
  CbArgs k{};
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
  k.nblk = static_cast<int32_t>(plan->n_blocks);
  k.n_panels = static_cast<int32_t>((qv + 32 * CH - 1) / (32 * CH));
  k.valid_vec = static_cast<int32_t>(qv);
  k.gp = std::max(1, std::min(gp, k.n_panels));
  k.n_groups = (k.n_panels + k.gp - 1) / k.gp;
  k.nrem = static_cast<int32_t>(plan->n_rem);
  k.goff = s.goff;
  k.blk = static_cast<const int4*>(plan->d_blk);
  k.pat_nv = static_cast<const int32_t*>(plan->d_pat_nv);
  k.vals = plan->d_vals;
  k.pat_ptr = static_cast<const int32_t*>(plan->d_pat_ptr);
  k.items = static_cast<const int4*>(plan->d_items);
  k.rem = static_cast<const int32_t*>(plan->d_rem);
  for (int l = 0; l < 8; ++l) k.off[l] = plan->off[l];
  k.s0 = s.s0;
  k.s1 = s.s1;
  k.s2 = s.s2;
  k.s3 = s.s3;
  const int64_t total = plan->n_blocks * k.n_groups;
  if (total >= (int64_t{1} << 31)) return false;
  const int grid = static_cast<int>((total + kWarps / SP - 1) / (kWarps / SP));
  const int64_t width = qv * 2;  // fp64 words per row (vectors of 16 B)
  constexpr int kPE = 32 * CH * 2;
  const CUtensorMap tm_w = make_tensor_map_f64(s.gsrc, a->n_cols, width, k.ldg_b, R + MM - 1, kPE);
  const CUtensorMap tm_v = mode == StepMode::Step ? make_tensor_map_f64(s.vin, a->n_rows, width, k.ldg_b, R, kPE) : tm_w;
  const CUtensorMap tm_y = mode == StepMode::Step ? make_tensor_map_f64(s.yin, a->n_rows, width, k.ldy_b, R, kPE) : tm_w;
  auto run = [&](auto kern, uint32_t warp_bytes) {
    constexpr int kTasks = kWarps / SP;
    const size_t smem = ((kTasks * (S + 1) * 8) + 127) / 128 * 128 + static_cast<size_t>(kTasks) * warp_bytes;
    if (smem > 48 * 1024)
      ADP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    launch_pdl(ctx, kern, dim3(grid), dim3(NT), smem, k, tm_w, tm_v, tm_y);
  };
  switch (mode) {
    case StepMode::First: run(cheb_cube_kernel<F, CH, R, L, MM, S, 0, RP, MINB, SP, LAZY, NT>, cube_warp_smem<F, CH, R, MM, S, 0>()); break;
    case StepMode::Step: run(cheb_cube_kernel<F, CH, R, L, MM, S, 1, RP, MINB, SP, LAZY, NT>, cube_warp_smem<F, CH, R, MM, S, 1>()); break;
    case StepMode::Deg1: run(cheb_cube_kernel<F, CH, R, L, MM, S, 2, RP, MINB, SP, LAZY, NT>, cube_warp_smem<F, CH, R, MM, S, 2>()); break;
    case StepMode::Spmm: run(cheb_cube_kernel<F, CH, R, L, MM, S, 3, RP, MINB, SP, LAZY, NT>, cube_warp_smem<F, CH, R, MM, S, 3>()); break;
    case StepMode::SpmmAcc: run(cheb_cube_kernel<F, CH, R, L, MM, S, 4, RP, MINB, SP, LAZY, NT>, cube_warp_smem<F, CH, R, MM, S, 4>()); break;
  }
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
  return true;
}


}  // namespace

// Automatic choice for the full 64-vector panels of a long-row real stencil operator (config 4):
// 2 x 2 lines of 2 rows, 1 KB panels, 2 ring stages, 4-warp CTAs (tools/tune_step.py).
bool launch_cube_auto(adp_ctx* ctx, StepMode mode, const StepArgs& s, int64_t qv) {
  const adp_csr* a = s.a;
  if (!ctx->auto_cube || a->dtype != ADP_F64) return false;
  return a->rp64 ? launch_cube_cfg<RealC, 2, 2, 2, 2, 3, 2, int64_t, 4, 1, false, 128>(ctx, mode, s, qv, 1, 0.5)
                 : launch_cube_cfg<RealC, 2, 2, 2, 2, 3, 2, int32_t, 4, 1, false, 128>(ctx, mode, s, qv, 1, 0.5);
}

bool launch_step_cube(adp_ctx* ctx, StepMode mode, const StepArgs& s) {
  // variant 4: the cube kernel forced on any real operator (its automatic geometry, no regularity floor)
  const adp_csr* a = s.a;
  if (ctx->variant != 4 || a->dtype != ADP_F64 || a->n_rows >= (int64_t{1} << 30)) return false;
  const int64_t qv = (s.q + 1) / 2;
  for (int64_t ld : {s.ld, s.ld_y, s.ld_out})
    if (ld % 2 != 0 || (ld / 2) * 16 >= (int64_t{1} << 32)) return false;
  return a->rp64 ? launch_cube_cfg<RealC, 2, 2, 2, 2, 3, 2, int64_t, 4, 1, false, 128>(ctx, mode, s, qv, 1, 0.0)
                 : launch_cube_cfg<RealC, 2, 2, 2, 2, 3, 2, int32_t, 4, 1, false, 128>(ctx, mode, s, qv, 1, 0.0);
}

}  // namespace adp
