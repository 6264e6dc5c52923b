// Row-tile preprocessing for the TMA-pipelined Clenshaw step kernel.
//
// The B200 counterpart of the reference's csr_to_tiled
// (proj/include/adapoly/tiled_matrix.hpp:58-94): rows are grouped into tiles
// (row blocks) and each tile lists the DISTINCT columns its rows touch -- the
// reference's "column segments" -- so the kernel fetches every needed W row
// panel once per tile into shared memory (one TMA bulk copy each) instead of
// once per nonzero. Tile height is chosen per tile so that the tile's distinct
// W rows plus its V / Y rows fit one shared-memory pipeline stage.
//
// Per tile the kernel also bulk-copies a metadata blob:
//   int32 rowoff[R+1]   entry offsets of the tile's rows (relative)
//   int32 own[R]        slot of the row's own column (r), or -1
//   (pad to 16 B)
//   int32 slot[nnz_t]   per entry (CSR order): index into the distinct list
//   (pad to 16 B)
//   value vals[nnz_t]   the CSR values (8 or 16 B each)
// Accumulation order inside a row stays the CSR order (ascending column), so
// results remain bit-identical to the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "adp_internal.hpp"

namespace adp {

namespace {
inline int64_t pad16(int64_t b) { return (b + 15) & ~int64_t{15}; }
}  // namespace

int64_t tile_blob_bytes(int64_t rows, int64_t nnz_t, int64_t val_bytes) {
  return pad16(4 * (2 * rows + 1)) + pad16(4 * nnz_t) + pad16(nnz_t * val_bytes);
}

const Tiling* get_tiling(adp_csr* a, int64_t panel_bytes, int64_t stage_bytes) {
  for (auto& t : a->tilings)
    if (t->panel_bytes == panel_bytes && t->stage_bytes == stage_bytes) return t->ok ? t.get() : nullptr;
  auto t = std::make_unique<Tiling>();
  t->panel_bytes = panel_bytes;
  t->stage_bytes = stage_bytes;
  const int64_t n = a->n_rows;
  const int64_t vb = a->dtype == ADP_C128 ? 16 : 8;
  ensure_host_copy(a);
  const std::vector<int64_t>& rp = a->h_row_ptr;
  const std::vector<int32_t>& ci = a->h_col;
  std::vector<int32_t> tile_row{0};
  std::vector<int64_t> tile_dptr{0}, tile_blob{0};
  std::vector<int32_t> dcol;
  std::vector<int32_t> mark(static_cast<size_t>(a->n_cols), -1), slot_of(static_cast<size_t>(a->n_cols), -1);
  bool ok = true;
  int64_t r = 0;
  int32_t tid = 0;
  std::vector<int32_t> cols;
  while (r < n) {
    const int64_t r0 = r;
    int64_t d = 0;
    cols.clear();
    while (r < n && r - r0 < kMaxTileRows) {
      int64_t add = 0;
      for (int64_t k = rp[r]; k < rp[r + 1]; ++k) add += mark[ci[k]] != tid;
      // a column may repeat only across rows, never within one (strictly increasing)
      const int64_t rows = r - r0 + 1;
      const int64_t nnz_t = rp[r + 1] - rp[r0];
      const int64_t need = tile_blob_bytes(rows, nnz_t, vb) + (d + add + 2 * rows) * panel_bytes;
      if (need > stage_bytes || d + add > kMaxTileDistinct) break;
      for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
        if (mark[ci[k]] != tid) {
          mark[ci[k]] = tid;
          cols.push_back(ci[k]);
        }
      }
      d += add;
      ++r;
    }
    if (r == r0) {  // a single row does not fit one stage: this panel width cannot be tiled
      ok = false;
      break;
    }
    std::sort(cols.begin(), cols.end());
    tile_row.push_back(static_cast<int32_t>(r));
    dcol.insert(dcol.end(), cols.begin(), cols.end());
    tile_dptr.push_back(static_cast<int64_t>(dcol.size()));
    tile_blob.push_back(tile_blob.back() + tile_blob_bytes(r - r0, rp[r] - rp[r0], vb));
    ++tid;
  }
  t->ok = ok;
  if (!ok) {
    a->tilings.push_back(std::move(t));
    return nullptr;
  }
  const int64_t T = static_cast<int64_t>(tile_row.size()) - 1;
  t->n_tiles = T;
  std::vector<uint8_t> blob(static_cast<size_t>(tile_blob.back()));
  int64_t max_rows = 0;
  for (int64_t ti = 0; ti < T; ++ti) {
    const int64_t r0 = tile_row[ti], r1 = tile_row[ti + 1], rows = r1 - r0;
    max_rows = std::max(max_rows, rows);
    const int64_t e0 = rp[r0], nnz_t = rp[r1] - e0;
    for (int64_t s = tile_dptr[ti]; s < tile_dptr[ti + 1]; ++s) slot_of[dcol[s]] = static_cast<int32_t>(s - tile_dptr[ti]);
    uint8_t* base = blob.data() + tile_blob[ti];
    auto* rowoff = reinterpret_cast<int32_t*>(base);
    int32_t* own = rowoff + rows + 1;
    for (int64_t j = 0; j <= rows; ++j) rowoff[j] = static_cast<int32_t>(rp[r0 + j] - e0);
    for (int64_t j = 0; j < rows; ++j) {
      own[j] = -1;
      const int64_t rr = r0 + j;
      if (rr < a->n_cols && slot_of[rr] >= 0) {
        // own column present among this tile's distinct columns?
        const int32_t s = slot_of[rr];
        if (s < tile_dptr[ti + 1] - tile_dptr[ti] && dcol[tile_dptr[ti] + s] == rr) own[j] = s;
      }
    }
    auto* slots = reinterpret_cast<int32_t*>(base + pad16(4 * (2 * rows + 1)));
    for (int64_t k = 0; k < nnz_t; ++k) slots[k] = slot_of[ci[e0 + k]];
    uint8_t* vals = base + pad16(4 * (2 * rows + 1)) + pad16(4 * nnz_t);
    std::memcpy(vals, static_cast<const uint8_t*>(a->h_values) + e0 * vb, static_cast<size_t>(nnz_t * vb));
    for (int64_t s = tile_dptr[ti]; s < tile_dptr[ti + 1]; ++s) slot_of[dcol[s]] = -1;
  }
  t->max_rows = max_rows;
  ADP_CUDA(cudaSetDevice(a->ctx->device));
  auto up = [&](void** dst, const void* src, size_t bytes) {
    ADP_CUDA(cudaMalloc(dst, std::max<size_t>(bytes, 16)));
    if (bytes) ADP_CUDA(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  };
  up(&t->d_tile_row, tile_row.data(), tile_row.size() * 4);
  up(&t->d_tile_dptr, tile_dptr.data(), tile_dptr.size() * 8);
  up(&t->d_tile_blob, tile_blob.data(), tile_blob.size() * 8);
  up(&t->d_dcol, dcol.data(), dcol.size() * 4);
  up(&t->d_blob, blob.data(), blob.size());
  t->distinct = static_cast<int64_t>(dcol.size());
  plan_uploads_done();
  a->tilings.push_back(std::move(t));
  return a->tilings.back().get();
}

Tiling::~Tiling() {
  cudaFree(d_tile_row);
  cudaFree(d_tile_dptr);
  cudaFree(d_tile_blob);
  cudaFree(d_dcol);
  cudaFree(d_blob);
}

}  // namespace adp
