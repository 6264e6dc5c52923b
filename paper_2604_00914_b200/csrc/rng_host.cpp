// Host Philox4x32-10 draws (product path): the seeded inputs of the solver
// (initial basis, trace probes, Lanczos start, top-up) and of the synthetic
// configuration generators. Restates proj/include/adapoly/philox.hpp:18-109 so
// seeded blocks are bit-identical to the reference's.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <thread>
#include <vector>

#include "adp_internal.hpp"

namespace {

struct Philox {
  uint32_t key0, key1;
  uint64_t stream;
  Philox(uint64_t seed, uint64_t s)
      : key0(static_cast<uint32_t>(seed)), key1(static_cast<uint32_t>(seed >> 32)), stream(s) {}
  void block(uint64_t counter, uint32_t out[4]) const {
    uint32_t c0 = static_cast<uint32_t>(counter), c1 = static_cast<uint32_t>(counter >> 32);
    uint32_t c2 = static_cast<uint32_t>(stream), c3 = static_cast<uint32_t>(stream >> 32);
    uint32_t k0 = key0, k1 = key1;
    for (int round = 0; round < 10; ++round) {
      if (round) {
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
      }
      const uint64_t p0 = uint64_t{0xD2511F53u} * c0;
      const uint64_t p1 = uint64_t{0xCD9E8D57u} * c2;
      const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
      const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
      c1 = static_cast<uint32_t>(p1);
      c3 = static_cast<uint32_t>(p0);
      c0 = n0;
      c2 = n2;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
  }
  uint32_t word(uint64_t i) const {
    uint32_t b[4];
    block(i / 4, b);
    return b[i % 4];
  }
  double gaussian(uint64_t i) const {
    uint32_t b[4];
    block(i / 4, b);
    const unsigned pair = static_cast<unsigned>((i % 4) / 2);
    const double u1 = (static_cast<double>(b[2 * pair]) + 0.5) * 0x1p-32;
    const double u2 = (static_cast<double>(b[2 * pair + 1]) + 0.5) * 0x1p-32;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 2.0 * std::numbers::pi * u2;
    return (i % 2 == 0) ? r * std::cos(t) : r * std::sin(t);
  }
};

// Draw i depends on i alone (counter-based), so blocks of the index range can be
// filled by independent threads with bit-identical results; chunks start on
// multiples of 4 so each Philox block is computed once.
template <class Fn>
void parallel_range(int64_t total, Fn fn) {
  const int64_t kMin = int64_t{1} << 16;
  const int64_t hw = std::max<int64_t>(1, std::min<int64_t>(32, std::thread::hardware_concurrency()));
  const int64_t nt = std::min<int64_t>(hw, (total + kMin - 1) / kMin);
  if (nt <= 1) {
    fn(int64_t{0}, total);
    return;
  }
  const int64_t chunk = ((total + nt - 1) / nt + 3) / 4 * 4;
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t b = t * chunk, e = std::min(total, b + chunk);
    if (b < e) th.emplace_back(fn, b, e);
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

// Column-major n x q block: element (r, c) is draw c * n + r (philox.hpp:96-98),
// i.e. draw i lands at out[i].
adp_status adp_fill_gaussian(double* out, int64_t n, int64_t q, uint64_t seed, uint64_t stream) {
  const Philox rng(seed, stream);
  parallel_range(n * q, [&](int64_t b, int64_t e) {
    int64_t i = b;
    while (i < e) {
      uint32_t w[4];
      rng.block(static_cast<uint64_t>(i) / 4, w);
      for (int64_t j = i; j < std::min(e, (i / 4 + 1) * 4); ++j) {
        const unsigned pair = static_cast<unsigned>((j % 4) / 2);
        const double u1 = (static_cast<double>(w[2 * pair]) + 0.5) * 0x1p-32;
        const double u2 = (static_cast<double>(w[2 * pair + 1]) + 0.5) * 0x1p-32;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double t = 2.0 * std::numbers::pi * u2;
        out[j] = (j % 2 == 0) ? r * std::cos(t) : r * std::sin(t);
      }
      i = (i / 4 + 1) * 4;
    }
  });
  return ADP_OK;
}

adp_status adp_fill_rademacher(double* out, int64_t n, int64_t q, uint64_t seed, uint64_t stream) {
  const Philox rng(seed, stream);
  parallel_range(n * q, [&](int64_t b, int64_t e) {
    int64_t i = b;
    while (i < e) {
      uint32_t w[4];
      rng.block(static_cast<uint64_t>(i) / 4, w);
      for (int64_t j = i; j < std::min(e, (i / 4 + 1) * 4); ++j) out[j] = (w[j % 4] >> 31) != 0 ? 1.0 : -1.0;
      i = (i / 4 + 1) * 4;
    }
  });
  return ADP_OK;
}

adp_status adp_philox_gaussian(uint64_t seed, uint64_t stream, uint64_t first, int64_t count, double* out) {
  const Philox rng(seed, stream);
  for (int64_t i = 0; i < count; ++i) out[i] = rng.gaussian(first + static_cast<uint64_t>(i));
  return ADP_OK;
}

adp_status adp_philox_uniform(uint64_t seed, uint64_t stream, uint64_t first, int64_t count, double* out) {
  const Philox rng(seed, stream);
  for (int64_t i = 0; i < count; ++i)
    out[i] = (static_cast<double>(rng.word(first + static_cast<uint64_t>(i))) + 0.5) * 0x1p-32;
  return ADP_OK;
}

adp_status adp_philox_block(uint64_t seed, uint64_t stream, uint64_t counter, uint32_t* out) {
  Philox(seed, stream).block(counter, out);
  return ADP_OK;
}

}  // extern "C"
