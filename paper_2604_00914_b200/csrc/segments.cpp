// Column-segment layout of R-row blocks for cheb_seg_kernel (cheb_seg.cu).
//
// The reference regroups CSR into row blocks of T_i rows whose entries are
// sorted into column segments (csr_to_tiled, proj/include/adapoly/
// tiled_matrix.hpp:58-94) so that every distinct B row is loaded once per block
// (maspmm, :194-209). This is the same regrouping for GPU warps with T_i = R:
// per block the ascending distinct columns, a row bitmask and R values per
// distinct column (zero where the row lacks it; masked off in the kernel). A
// row still meets its own entries in ascending column order, so the kernel's
// per-element accumulation order -- and its bits -- are the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

Segments::~Segments() {
  cudaFree(d_blk_ptr);
  cudaFree(d_col);
  cudaFree(d_mask);
  cudaFree(d_val);
}

const Segments* get_segments(adp_csr* a, int R) {
  for (auto& s : a->segments)
    if (s->rows_per_block == R) return s.get();
  if (R < 1 || R > 32) fail(ADP_ERR_CONFIG, "segments: rows per block must be in [1, 32]");
  auto s = std::make_unique<Segments>();
  s->rows_per_block = R;
  const int64_t n = a->n_rows;
  const int64_t vb = a->dtype == ADP_C128 ? 16 : 8;
  const int64_t nb = (n + R - 1) / R;
  ensure_host_copy(a);
  const std::vector<int64_t>& rp = a->h_row_ptr;
  const std::vector<int32_t>& ci = a->h_col;
  const auto* hv = static_cast<const uint8_t*>(a->h_values);
  std::vector<int64_t> blk_ptr(nb + 1, 0);
  // pass 1: count distinct columns per block (R-way merge of sorted rows)
  std::vector<int64_t> cur(R), end(R);
  auto walk = [&](int64_t b, auto&& emit) {
    const int64_t r0 = b * R;
    const int rows = static_cast<int>(std::min<int64_t>(R, n - r0));
    for (int i = 0; i < rows; ++i) {
      cur[i] = rp[r0 + i];
      end[i] = rp[r0 + i + 1];
    }
    while (true) {
      int32_t c = INT32_MAX;
      for (int i = 0; i < rows; ++i)
        if (cur[i] < end[i]) c = std::min(c, ci[cur[i]]);
      if (c == INT32_MAX) break;
      uint32_t mask = 0;
      int64_t idx[32];
      for (int i = 0; i < rows; ++i) {
        idx[i] = -1;
        if (cur[i] < end[i] && ci[cur[i]] == c) {
          mask |= 1u << i;
          idx[i] = cur[i]++;
        }
      }
      emit(c, mask, idx, rows);
    }
  };
  for (int64_t b = 0; b < nb; ++b) {
    int64_t cnt = 0;
    walk(b, [&](int32_t, uint32_t, const int64_t*, int) { ++cnt; });
    blk_ptr[b + 1] = blk_ptr[b] + cnt;
  }
  const int64_t S = blk_ptr[nb];
  std::vector<int32_t> col(static_cast<size_t>(S));
  std::vector<uint32_t> msk(static_cast<size_t>(S));
  std::vector<uint8_t> val(static_cast<size_t>(S * R * vb), 0);
  for (int64_t b = 0; b < nb; ++b) {
    int64_t sidx = blk_ptr[b];
    walk(b, [&](int32_t c, uint32_t mask, const int64_t* idx, int rows) {
      col[sidx] = c;
      msk[sidx] = mask;
      for (int i = 0; i < rows; ++i)
        if (idx[i] >= 0) std::memcpy(&val[(sidx * R + i) * vb], hv + idx[i] * vb, static_cast<size_t>(vb));
      ++sidx;
    });
  }
  s->n_blocks = nb;
  s->n_segs = S;
  s->reuse = S > 0 ? static_cast<double>(a->nnz) / static_cast<double>(S) : 1.0;
  ADP_CUDA(cudaSetDevice(a->ctx->device));
  auto up = [&](void** dst, const void* src, size_t bytes) {
    ADP_CUDA(cudaMalloc(dst, std::max<size_t>(bytes, 16)));
    if (bytes) ADP_CUDA(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  };
  up(&s->d_blk_ptr, blk_ptr.data(), blk_ptr.size() * 8);
  up(&s->d_col, col.data(), col.size() * 4);
  up(&s->d_mask, msk.data(), msk.size() * 4);
  up(&s->d_val, val.data(), val.size());
  plan_uploads_done();
  a->segments.push_back(std::move(s));
  return a->segments.back().get();
}

}  // namespace adp
