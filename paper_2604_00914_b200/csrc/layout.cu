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

#include <cstdint>

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

}  // namespace adp
