// The INTEGRATION.md binding compiled against the REFERENCE's own headers and sources (proj/include,
// proj/src/cheb_filter.cpp, in place under /root/reference; Eigen replaced by oracle/eigen_standin) and run
// the way a reference test would: the reference's CPU clenshaw_apply / maspmm against gpu::clenshaw_apply /
// gpu::maspmm on operators built with the reference's from_triplets and blocks from its Philox fills.
// Bitwise equality, the spmv accounting and the exception types are checked. Test infrastructure.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "adapoly/cheb_filter.hpp"
#include "adapoly/csr_matrix.hpp"
#include "adapoly/philox.hpp"
#include "adapoly/tiled_matrix.hpp"
#include "adapoly_gpu_shim.hpp"

using namespace adapoly;

namespace {
std::uint64_t lcg(std::uint64_t& s) { return s = s * 6364136223846793005ull + 1442695040888963407ull; }
double unit(std::uint64_t& s) { return static_cast<double>(lcg(s) >> 11) * 0x1p-53; }

CsrMatrixd random_symmetric(index_t n, double density, std::uint64_t seed) {
  std::vector<Triplet<double>> t;
  for (index_t i = 0; i < n; ++i) {
    t.push_back({i, i, 2.0 * unit(seed) - 1.0});
    for (index_t j = i + 1; j < n; ++j)
      if (unit(seed) < density) {
        const double v = 2.0 * unit(seed) - 1.0;
        t.push_back({i, j, v});
        t.push_back({j, i, v});
      }
  }
  return CsrMatrixd::from_triplets(n, n, t);
}

// 7-point Laplacian + diagonal potential on an nx x ny x nz grid: takes the plane-sweep kernel on the GPU
CsrMatrixd stencil7(index_t nx, index_t ny, index_t nz, std::uint64_t seed) {
  std::vector<Triplet<double>> t;
  const index_t n = nx * ny * nz;
  for (index_t r = 0; r < n; ++r) {
    const index_t x = r % nx, y = (r / nx) % ny, z = r / (nx * ny);
    t.push_back({r, r, 6.0 + 4.0 * unit(seed) - 2.0});
    if (x > 0) t.push_back({r, r - 1, -1.0});
    if (x < nx - 1) t.push_back({r, r + 1, -1.0});
    if (y > 0) t.push_back({r, r - nx, -1.0});
    if (y < ny - 1) t.push_back({r, r + nx, -1.0});
    if (z > 0) t.push_back({r, r - nx * ny, -1.0});
    if (z < nz - 1) t.push_back({r, r + nx * ny, -1.0});
  }
  return CsrMatrixd::from_triplets(n, n, t);
}

bool same(const Matrixd& a, const Matrixd& b) {
  return a.rows() == b.rows() && a.cols() == b.cols() &&
         std::memcmp(a.data(), b.data(), sizeof(double) * static_cast<std::size_t>(a.rows() * a.cols())) == 0;
}
}  // namespace

int main() {
  gpu::Device dev(0);
  int cases = 0;
  struct Op {
    CsrMatrixd a;
    SpectrumBounds b;
    double lo, hi;
  };
  std::vector<Op> ops;
  ops.push_back({random_symmetric(300, 0.04, 7), {-12.0, 12.0}, -2.0, 1.5});
  ops.push_back({stencil7(12, 10, 9, 3), {-2.0, 14.0}, 5.5, 6.5});
  for (const Op& op : ops) {
    const CsrMatrixd& a = op.a;
    a.validate();
    const TiledMatrixd tiled = csr_to_tiled(a, default_tile_ti, default_tile_tk);
    gpu::DeviceMatrix dmat(dev, a);
    const ChebFilter f = build_filter(op.lo, op.hi, op.b, 40, 0.5);
    for (index_t q : {index_t{1}, index_t{5}, index_t{64}, index_t{70}}) {
      Matrixd x(a.n_rows, q);
      fill_gaussian(x, 11 + static_cast<std::uint64_t>(q), 0);
      for (int degree : {0, 1, 2, 7, 40}) {
        std::int64_t c_cpu = 0, c_gpu = 0;
        const Matrixd want = clenshaw_apply(f, tiled, x, degree, &c_cpu);
        const Matrixd got = gpu::clenshaw_apply(dev, f, dmat, x, degree, &c_gpu);
        if (!same(got, want) || c_cpu != c_gpu) {
          std::printf("MISMATCH n=%lld q=%lld degree=%d (spmv %lld vs %lld)\n", static_cast<long long>(a.n_rows),
                      static_cast<long long>(q), degree, static_cast<long long>(c_cpu), static_cast<long long>(c_gpu));
          return 1;
        }
        ++cases;
      }
      // maspmm: C += A B through the reference's block layout vs the shim
      Matrixd b(a.n_cols, q), c0(a.n_rows, q);
      fill_gaussian(b, 5, 1);
      fill_gaussian(c0, 6, 2);
      BlockMatrixd bb = to_block_layout<double>(b, default_tile_tk), cb = to_block_layout<double>(c0, default_tile_tk);
      maspmm(tiled, bb, cb);
      Matrixd cg = c0;
      gpu::maspmm(dev, dmat, b, cg);
      if (!same(cg, from_block_layout(cb))) {
        std::printf("MISMATCH maspmm n=%lld q=%lld\n", static_cast<long long>(a.n_rows), static_cast<long long>(q));
        return 1;
      }
      ++cases;
    }
    // the reference's exception types come back through the status mapping
    Matrixd x(a.n_rows, 3);
    fill_gaussian(x, 1, 0);
    bool threw = false;
    try {
      gpu::clenshaw_apply(dev, f, dmat, x, 41);
    } catch (const ConfigError&) {
      threw = true;
    }
    Matrixd bad(a.n_rows - 1, 3);
    bool threw2 = false;
    try {
      gpu::clenshaw_apply(dev, f, dmat, bad, 3);
    } catch (const DimensionError&) {
      threw2 = true;
    }
    if (!threw || !threw2) {
      std::printf("exception mapping failed\n");
      return 1;
    }
  }
  std::printf("reference shim: %d cases bitwise==reference, exceptions mapped\n", cases);
  return 0;
}
