// Layout conversion and seeded-fill kernels.
//
// The reference converts Eigen column-major blocks to its row-segment layout
// and back once per clenshaw_apply call (to_block_layout / from_block_layout,
// proj/include/adapoly/tiled_matrix.hpp:151-175). On the device the dense
// operands are plain row-major n x q (what BlockMatrix degenerates to when
// t_k >= q), so the only conversions are the column-major <-> row-major
// transposes at the host boundary: 32x32 shared-memory tiles, coalesced on
// both sides. Pure data movement -- bitwise exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <new>
#include <vector>

#include "adp_internal.hpp"

namespace adp {
namespace {

constexpr int kTile = 32;
constexpr int kRowsPerIter = 8;

// dst[r * ldd + c] = src[c * lds + r]   (col-major n x q  ->  row-major n x q)
template <class T>
__global__ void col_to_row_kernel(const T* __restrict__ src, int64_t n, int64_t q, int64_t lds, T* __restrict__ dst,
                                  int64_t ldd) {
  __shared__ T tile[kTile][kTile + 1];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * kTile;
  // read: consecutive threads walk rows (contiguous in column-major)
  for (int j = threadIdx.y; j < kTile; j += kRowsPerIter) {
    const int64_t c = c0 + j, r = r0 + threadIdx.x;
    if (c < q && r < n) tile[j][threadIdx.x] = src[c * lds + r];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < kTile; j += kRowsPerIter) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    if (r < n && c < q) dst[r * ldd + c] = tile[threadIdx.x][j];
  }
}

// dst[c * ldd + r] = src[r * lds + c]   (row-major n x q  ->  col-major n x q)
template <class T>
__global__ void row_to_col_kernel(const T* __restrict__ src, int64_t n, int64_t q, int64_t lds, T* __restrict__ dst,
                                  int64_t ldd) {
  __shared__ T tile[kTile][kTile + 1];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * kTile;
  for (int j = threadIdx.y; j < kTile; j += kRowsPerIter) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    if (r < n && c < q) tile[j][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < kTile; j += kRowsPerIter) {
    const int64_t c = c0 + j, r = r0 + threadIdx.x;
    if (c < q && r < n) dst[c * ldd + r] = tile[threadIdx.x][j];
  }
}

// dst row-major = s * src row-major (componentwise for complex).
__global__ void scale_rows_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                                  int64_t n, int64_t qd, double s) {
  const int64_t total = n * qd;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / qd, c = i - r * qd;
    dst[r * ldd + c] = __dmul_rn(s, src[r * lds + c]);
  }
}

// Philox4x32-10 (proj/include/adapoly/philox.hpp:25-51), device side.
__device__ __forceinline__ uint4 philox_block(uint64_t seed, uint64_t stream, uint64_t counter) {
  uint32_t c0 = static_cast<uint32_t>(counter), c1 = static_cast<uint32_t>(counter >> 32);
  uint32_t c2 = static_cast<uint32_t>(stream), c3 = static_cast<uint32_t>(stream >> 32);
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round != 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}

// kind 0: gaussian (Box-Muller, philox.hpp:59-67; device libm, so last-ulp
// differences vs glibc are possible), kind 1: rademacher (exact, :70-72).
// Draw index c*n + r (column-major storage order, :96-98), stored row-major.
__global__ void fill_philox_kernel(double* dst, int64_t n, int64_t q, int64_t ld, uint64_t seed, uint64_t stream,
                                   int kind) {
  const int64_t total = n * q;
  // walk the storage (row-major) order so the writes coalesce; the draw index
  // is still the reference's column-major c*n + r
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < total;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = s / q, c = s - r * q;
    const uint64_t idx = static_cast<uint64_t>(c * n + r);
    const uint4 b = philox_block(seed, stream, idx / 4);
    const uint32_t w[4] = {b.x, b.y, b.z, b.w};
    double v;
    if (kind == 1) {
      v = (w[idx % 4] >> 31) != 0 ? 1.0 : -1.0;
    } else {
      const int pair = static_cast<int>((idx % 4) / 2);
      const double u1 = (static_cast<double>(w[2 * pair]) + 0.5) * 0x1p-32;
      const double u2 = (static_cast<double>(w[2 * pair + 1]) + 0.5) * 0x1p-32;
      const double rr = sqrt(-2.0 * log(u1));
      const double t = 2.0 * 3.141592653589793 * u2;
      v = (idx % 2 == 0) ? rr * cos(t) : rr * sin(t);
    }
    dst[r * ld + c] = v;
  }
}

int grid_for(adp_ctx* ctx, int64_t total, int threads) {
  const int64_t want = (total + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 8;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

void launch_colmajor_to_rowmajor(adp_ctx* ctx, const void* src, int64_t n, int64_t q, int64_t lds, void* dst,
                                 int64_t ldd, int elem_bytes) {
  if (n == 0 || q == 0) return;
  const dim3 grid(static_cast<unsigned>((n + kTile - 1) / kTile), static_cast<unsigned>((q + kTile - 1) / kTile));
  const dim3 block(kTile, kRowsPerIter);
  if (elem_bytes == 8)
    col_to_row_kernel<double><<<grid, block, 0, ctx->stream>>>(static_cast<const double*>(src), n, q, lds,
                                                               static_cast<double*>(dst), ldd);
  else
    col_to_row_kernel<double2><<<grid, block, 0, ctx->stream>>>(static_cast<const double2*>(src), n, q, lds,
                                                                static_cast<double2*>(dst), ldd);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

void launch_rowmajor_to_colmajor(adp_ctx* ctx, const void* src, int64_t n, int64_t q, int64_t lds, void* dst,
                                 int64_t ldd, int elem_bytes) {
  if (n == 0 || q == 0) return;
  const dim3 grid(static_cast<unsigned>((n + kTile - 1) / kTile), static_cast<unsigned>((q + kTile - 1) / kTile));
  const dim3 block(kTile, kRowsPerIter);
  if (elem_bytes == 8)
    row_to_col_kernel<double><<<grid, block, 0, ctx->stream>>>(static_cast<const double*>(src), n, q, lds,
                                                               static_cast<double*>(dst), ldd);
  else
    row_to_col_kernel<double2><<<grid, block, 0, ctx->stream>>>(static_cast<const double2*>(src), n, q, lds,
                                                                static_cast<double2*>(dst), ldd);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

void launch_scale_rows(adp_ctx* ctx, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t n, int64_t q,
                       double s, int elem_bytes) {
  const int64_t f = elem_bytes / 8;  // doubles per element
  if (n == 0 || q == 0) return;
  scale_rows_kernel<<<grid_for(ctx, n * q * f, 256), 256, 0, ctx->stream>>>(
      static_cast<const double*>(src), lds * f, static_cast<double*>(dst), ldd * f, n, q * f, s);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

void launch_fill_philox(adp_ctx* ctx, double* dst, int64_t n, int64_t q, int64_t ld, uint64_t seed,
                        uint64_t stream, int kind) {
  if (n == 0 || q == 0) return;
  fill_philox_kernel<<<grid_for(ctx, n * q, 256), 256, 0, ctx->stream>>>(dst, n, q, ld, seed, stream, kind);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

// ---- device-side CSR checks (adp_csr_create_device) ---------------------------------------
namespace {

// One thread per row: bit 0 = row_ptr decreasing or endpoints wrong, bit 1 = column out of
// range, bit 2 = columns not strictly increasing (the CsrMatrix invariant, csr_matrix.hpp:101-116).
__global__ void validate_csr_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t n_rows,
                                    int64_t n_cols, int64_t nnz, int* __restrict__ flags) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int bad = 0;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows; r += stride) {
    const int64_t b = rp[r], e = rp[r + 1];
    if (e < b || b < 0 || e > nnz || (r == 0 && b != 0) || (r == n_rows - 1 && e != nnz)) {
      bad |= 1;
      continue;
    }
    int32_t prev = -1;
    for (int64_t k = b; k < e; ++k) {
      const int32_t c = col[k];
      if (c < 0 || c >= n_cols) bad |= 2;
      if (k > b && c <= prev) bad |= 4;
      prev = c;
    }
  }
  if (bad) atomicOr(flags, bad);
}

__global__ void narrow_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t count) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
    dst[i] = static_cast<int32_t>(src[i]);
}

}  // namespace

int validate_csr_device(adp_ctx* ctx, const int64_t* row_ptr, const int32_t* col, int64_t n_rows, int64_t n_cols,
                        int64_t nnz) {
  int* flags = nullptr;
  ADP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flags), sizeof(int), ctx->stream));
  ADP_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), ctx->stream));
  int h = 0;
  if (n_rows > 0) {
    validate_csr_kernel<<<grid_for(ctx, n_rows, 256), 256, 0, ctx->stream>>>(row_ptr, col, n_rows, n_cols, nnz, flags);
    ADP_LAUNCH_CHECK();
    ctx->launches += 1;
  }
  ADP_CUDA(cudaMemcpyAsync(&h, flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  ADP_CUDA(cudaFreeAsync(flags, ctx->stream));
  ADP_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

void narrow_row_ptr_device(adp_ctx* ctx, const int64_t* src, int32_t* dst, int64_t count) {
  if (count == 0) return;
  narrow_kernel<<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(src, dst, count);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

void ensure_host_copy(adp_csr* a) {
  if (a->host_ready) return;
  const size_t eb = a->dtype == ADP_C128 ? 16 : 8;
  ADP_CUDA(cudaSetDevice(a->device));
  ADP_CUDA(cudaDeviceSynchronize());
  a->h_row_ptr.resize(a->n_rows + 1);
  if (a->rp64) {
    ADP_CUDA(cudaMemcpy(a->h_row_ptr.data(), a->row_ptr, (a->n_rows + 1) * 8, cudaMemcpyDeviceToHost));
  } else {
    std::vector<int32_t> rp32(a->n_rows + 1);
    ADP_CUDA(cudaMemcpy(rp32.data(), a->row_ptr, (a->n_rows + 1) * 4, cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r <= a->n_rows; ++r) a->h_row_ptr[r] = rp32[r];
  }
  a->h_col.resize(a->nnz);
  void* hv = std::malloc(std::max<size_t>(a->nnz, 1) * eb);
  if (!hv) throw std::bad_alloc();
  if (a->nnz) {
    ADP_CUDA(cudaMemcpy(a->h_col.data(), a->col_idx, a->nnz * 4, cudaMemcpyDeviceToHost));
    ADP_CUDA(cudaMemcpy(hv, a->values, a->nnz * eb, cudaMemcpyDeviceToHost));
  }
  a->h_values = hv;
  a->host_ready = true;
}

// ---- halo exchange over peer memory (multi-GPU row partition) ------------------------------
namespace {

struct PushSet {
  PushTarget t[kMaxPush];
  int32_t n;
};

// One warp per (row, target): 16-byte coalesced copies of the row into the neighbour's halo.
__global__ void push_rows_kernel(const char* __restrict__ src, int64_t ld_b, int64_t row_begin, int64_t row_end,
                                 int64_t row_bytes, PushSet ps) {
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  const int lane = threadIdx.x % 32;
  bool wrote = false;
  for (int t = 0; t < ps.n; ++t) {
    const int64_t lo = max(row_begin, ps.t[t].lo), hi = min(row_end, ps.t[t].hi);
    for (int64_t r = lo + (static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32); r < hi; r += warps) {
      const int4* s4 = reinterpret_cast<const int4*>(src + r * ld_b);
      int4* d4 = reinterpret_cast<int4*>(ps.t[t].dst + static_cast<uint64_t>(r + ps.t[t].shift) * ps.t[t].ld_b);
      for (int64_t i = lane; i < row_bytes / 16; i += 32) d4[i] = s4[i];
      wrote = true;
    }
  }
  if (wrote) __threadfence_system();
}

struct CounterSet {
  uint64_t* c[kMaxPush];
  int32_t n;
};

__global__ void halo_signal_kernel(CounterSet cs, uint64_t value) {
  // every kernel before this one on the stream has retired, and each thread that stored to a peer
  // fenced at system scope first: the halo rows are visible to the peer before the counter moves
  asm volatile("fence.sc.sys;\n" ::: "memory");
  for (int i = 0; i < cs.n; ++i) asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(cs.c[i]), "l"(value) : "memory");
}

__global__ void halo_wait_kernel(CounterSet cs, uint64_t expected, uint64_t timeout_ns, int* failed) {
  if (*(volatile int*)failed) return;  // an earlier wait of this call timed out: fail fast, do not spin again
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < cs.n; ++i) {
    while (true) {
      uint64_t v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(cs.c[i]) : "memory");
      if (v >= expected) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {  // a neighbour that never signals: fail the step, do not hang the GPU
        *failed = 1;
        return;
      }
      __nanosleep(200);
    }
  }
}

}  // namespace

void launch_push_rows(adp_ctx* ctx, const void* src, int64_t ld_b, int64_t row_begin, int64_t row_end,
                      int64_t row_bytes, const PushTarget* targets, int32_t n) {
  if (n <= 0 || row_end <= row_begin) return;
  if (n > kMaxPush) fail(ADP_ERR_CONFIG, "halo push: too many targets");
  if (row_bytes % 16 || ld_b % 16 || (reinterpret_cast<uintptr_t>(src) & 15u))
    fail(ADP_ERR_DIMENSION, "halo push: rows must be 16-byte aligned");
  PushSet ps{};
  ps.n = n;
  int64_t rows = 0;
  for (int i = 0; i < n; ++i) {
    ps.t[i] = targets[i];
    if (ps.t[i].ld_b % 16 || (reinterpret_cast<uintptr_t>(ps.t[i].dst) & 15u))
      fail(ADP_ERR_DIMENSION, "halo push: target rows must be 16-byte aligned");
    rows += std::max<int64_t>(0, std::min(row_end, ps.t[i].hi) - std::max(row_begin, ps.t[i].lo));
  }
  if (rows == 0) return;
  push_rows_kernel<<<grid_for(ctx, rows * 32, 256), 256, 0, ctx->stream>>>(static_cast<const char*>(src), ld_b,
                                                                            row_begin, row_end, row_bytes, ps);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

void launch_halo_signal(adp_ctx* ctx, uint64_t* const* counters, int32_t n, uint64_t value) {
  if (n <= 0) return;
  if (n > kMaxPush) fail(ADP_ERR_CONFIG, "halo signal: too many counters");
  CounterSet cs{};
  cs.n = n;
  for (int i = 0; i < n; ++i) cs.c[i] = counters[i];
  halo_signal_kernel<<<1, 1, 0, ctx->stream>>>(cs, value);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

void launch_halo_wait(adp_ctx* ctx, const uint64_t* const* counters, int32_t n, uint64_t expected,
                      uint32_t timeout_ms) {
  if (n <= 0) return;
  if (n > kMaxPush) fail(ADP_ERR_CONFIG, "halo wait: too many counters");
  CounterSet cs{};
  cs.n = n;
  for (int i = 0; i < n; ++i) cs.c[i] = const_cast<uint64_t*>(counters[i]);
  if (!ctx->halo_failed) {  // fresh memory may hold stale bytes: clear before the first wait reads it
    ADP_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->halo_failed), sizeof(int)));
    ADP_CUDA(cudaMemsetAsync(ctx->halo_failed, 0, sizeof(int), ctx->stream));
  }
  halo_wait_kernel<<<1, 1, 0, ctx->stream>>>(cs, expected, static_cast<uint64_t>(timeout_ms) * 1000000ull,
                                             ctx->halo_failed);
  ADP_LAUNCH_CHECK();
  ctx->launches += 1;
}

}  // namespace adp
