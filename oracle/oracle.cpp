// ============================================================================
// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the AdaPolySI Chebyshev-filter hot path of the reference
// (/root/reference/proj, C++20 + Eigen + OpenMP). The reference as a whole
// cannot be compiled in this image (Eigen3 and vendor/ are absent, SURVEY.md
// 0.4), so this file restates, op for op, the functions on the path; the
// reference's own FILTER-PATH sources are compiled in place against a minimal
// Eigen stand-in into oracle/_ref (ref_capi.cpp, eigen_standin/), and
// tests/test_ref_build.py checks this restatement bit for bit against them. It is the
// CHECKER for the CUDA product path: only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it.
//
// Build recipe (oracle/Makefile): g++ -O3 -fopenmp -ffp-contract=off, with no
// -march, mirroring the reference Release build (proj/CMakeLists.txt:7-9), so
// the floating-point op sequence -- and therefore every bit -- matches the
// reference on x86-64 (SSE2, no FMA).
//
// Parity is pinned by the reference's own known-answer tests restated in
// tests/test_oracle_pins.py (proj/tests/test_cheb_filter.cpp,
// proj/tests/test_sparse_core.cpp, proj/tests/acceptance.cpp criteria 4/5/7),
// the Philox4x32-10 published known-answer vectors, and the reference's three
// .mtx fixtures (converted by tests/golden/make_golden.py).
//
// Complex (complex128) entry points have NO reference counterpart
// (SPEC.md:15,115); they are pinned by the real 2n x 2n embedding
// S = [[Re H, -Im H], [Im H, Re H]] against the real path.
// ============================================================================
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

using index_t = std::int64_t;
constexpr double pi = std::numbers::pi;

// ---------------------------------------------------------------- errors ---
// Status codes mirror the reference exception types (proj/include/adapoly/types.hpp:23-46).
enum Status { OK = 0, CONFIG = 1, DIMENSION = 2, NOT_PD = 3, PARSE = 4, RUNTIME = 5 };
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return RUNTIME;
    }
}

// --------------------------------------------------------------- scalars ---
// Minimal complex type with an explicit, fixed op order (the GPU kernels use
// the same order); the SpMM accumulation is mac() below.
struct cplx {
    double re, im;
};
inline cplx operator+(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
inline cplx operator-(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
inline cplx operator*(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline cplx operator*(double s, cplx a) { return {s * a.re, s * a.im}; }
inline cplx& operator+=(cplx& a, cplx b) { a = a + b; return a; }
// The SpMM accumulation c += v * b. Real: the reference's unfused multiply then add
// (tiled_matrix.hpp:205 under SSE2, no FMA). Complex has no reference:
// its accumulation is DEFINED as four fused multiply-adds in this order, which the GPU
// kernels use too (__fma_rn); it is pinned to the real path by the 2n x 2n embedding.
inline void mac(double& c, double v, double b) { c += v * b; }
inline void mac(cplx& c, cplx v, cplx b) {
    c.re = std::fma(v.re, b.re, c.re);
    c.re = std::fma(-v.im, b.im, c.re);
    c.im = std::fma(v.re, b.im, c.im);
    c.im = std::fma(v.im, b.re, c.im);
}

template <class S> inline S zero();
template <> inline double zero<double>() { return 0.0; }
template <> inline cplx zero<cplx>() { return {0.0, 0.0}; }

// ----------------------------------------------------------------- philox ---
// Philox4x32-10 (proj/include/adapoly/philox.hpp:18-80).
struct Philox {
    std::uint32_t key0, key1;
    std::uint64_t stream;
    Philox(std::uint64_t seed, std::uint64_t s)
        : key0(static_cast<std::uint32_t>(seed)), key1(static_cast<std::uint32_t>(seed >> 32)), stream(s) {}

    void block(std::uint64_t counter, std::uint32_t out[4]) const {  // philox.hpp:25-51
        std::uint32_t c0 = static_cast<std::uint32_t>(counter);
        std::uint32_t c1 = static_cast<std::uint32_t>(counter >> 32);
        std::uint32_t c2 = static_cast<std::uint32_t>(stream);
        std::uint32_t c3 = static_cast<std::uint32_t>(stream >> 32);
        std::uint32_t k0 = key0, k1 = key1;
        for (int round = 0; round < 10; ++round) {
            if (round != 0) {
                k0 += 0x9E3779B9u;
                k1 += 0xBB67AE85u;
            }
            const std::uint64_t p0 = std::uint64_t{0xD2511F53u} * c0;
            const std::uint64_t p1 = std::uint64_t{0xCD9E8D57u} * c2;
            const std::uint32_t n0 = static_cast<std::uint32_t>(p1 >> 32) ^ c1 ^ k0;
            const std::uint32_t n2 = static_cast<std::uint32_t>(p0 >> 32) ^ c3 ^ k1;
            c1 = static_cast<std::uint32_t>(p1);
            c3 = static_cast<std::uint32_t>(p0);
            c0 = n0;
            c2 = n2;
        }
        out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
    }
    std::uint32_t word(std::uint64_t i) const {
        std::uint32_t b[4];
        block(i / 4, b);
        return b[i % 4];
    }
    double gaussian(std::uint64_t i) const {  // philox.hpp:59-67
        std::uint32_t b[4];
        block(i / 4, b);
        const std::size_t pair = (i % 4) / 2;
        const double u1 = (static_cast<double>(b[2 * pair]) + 0.5) * 0x1p-32;
        const double u2 = (static_cast<double>(b[2 * pair + 1]) + 0.5) * 0x1p-32;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double t = 2.0 * pi * u2;
        return (i % 2 == 0) ? r * std::cos(t) : r * std::sin(t);
    }
    double rademacher(std::uint64_t i) const { return (word(i) >> 31) != 0 ? 1.0 : -1.0; }  // :70-72
    double uniform(std::uint64_t i) const { return (static_cast<double>(word(i)) + 0.5) * 0x1p-32; }
};

// -------------------------------------------------------------------- csr ---
template <class S>
struct Csr {
    index_t n_rows = 0, n_cols = 0;
    std::vector<index_t> row_ptr{0}, col_idx;
    std::vector<S> values;
    index_t nnz() const { return static_cast<index_t>(values.size()); }
};

template <class S>
struct Triplet {
    index_t row, col;
    S value;
};

// CsrMatrix::from_triplets (proj/include/adapoly/csr_matrix.hpp:34-62): sort by
// (row, col), sum duplicates in sorted order.
template <class S>
Csr<S> from_triplets(index_t rows, index_t cols, std::vector<Triplet<S>> entries) {
    if (rows < 0 || cols < 0) throw Error(DIMENSION, "negative matrix size");
    std::sort(entries.begin(), entries.end(), [](const Triplet<S>& a, const Triplet<S>& b) {
        return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    Csr<S> m;
    m.n_rows = rows;
    m.n_cols = cols;
    m.row_ptr.assign(static_cast<std::size_t>(rows) + 1, 0);
    for (std::size_t i = 0; i < entries.size();) {
        const index_t r = entries[i].row, c = entries[i].col;
        if (r < 0 || r >= rows || c < 0 || c >= cols) throw Error(DIMENSION, "triplet index out of bounds");
        S v = entries[i].value;
        for (++i; i < entries.size() && entries[i].row == r && entries[i].col == c; ++i) v += entries[i].value;
        m.col_idx.push_back(c);
        m.values.push_back(v);
        ++m.row_ptr[static_cast<std::size_t>(r) + 1];
    }
    for (index_t r = 0; r < rows; ++r) m.row_ptr[r + 1] += m.row_ptr[r];
    return m;
}

// --------------------------------------------------------------- tiled -----
// TiledMatrix + csr_to_tiled (proj/include/adapoly/tiled_matrix.hpp:23-94).
template <class S>
struct Tiled {
    index_t n_rows = 0, n_cols = 0, t_i = 0, t_k = 0;
    std::vector<index_t> act_colseg{0}, colseg_ptr{0}, col_idx, row_idx;
    std::vector<S> values;
    index_t row_blocks() const { return t_i > 0 ? (n_rows + t_i - 1) / t_i : 0; }
};

template <class S>
Tiled<S> csr_to_tiled(const Csr<S>& a, index_t t_i, index_t t_k) {
    if (t_i < 1 || t_k < 1) throw Error(CONFIG, "csr_to_tiled: tile sizes must be >= 1");
    Tiled<S> t;
    t.n_rows = a.n_rows;
    t.n_cols = a.n_cols;
    t.t_i = t_i;
    t.t_k = t_k;
    t.row_idx.reserve(a.values.size());
    t.values.reserve(a.values.size());
    std::vector<Triplet<S>> be;
    for (index_t ib = 0; ib < t.row_blocks(); ++ib) {
        const index_t lo = ib * t_i, hi = std::min(lo + t_i, a.n_rows);
        be.clear();
        for (index_t r = lo; r < hi; ++r)
            for (index_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) be.push_back({r, a.col_idx[k], a.values[k]});
        std::sort(be.begin(), be.end(), [](const Triplet<S>& x, const Triplet<S>& y) {
            return x.col != y.col ? x.col < y.col : x.row < y.row;
        });
        for (std::size_t i = 0; i < be.size();) {
            const index_t col = be[i].col;
            t.col_idx.push_back(col);
            for (; i < be.size() && be[i].col == col; ++i) {
                t.row_idx.push_back(be[i].row);
                t.values.push_back(be[i].value);
            }
            t.colseg_ptr.push_back(static_cast<index_t>(t.values.size()));
        }
        t.act_colseg.push_back(static_cast<index_t>(t.col_idx.size()));
    }
    return t;
}

// BlockMatrix (tiled_matrix.hpp:100-147): column blocks of width t_k, each a
// contiguous row-major rows x width panel.
template <class S>
struct Block {
    index_t rows = 0, cols = 0, t_k = 1;
    std::vector<index_t> offsets{0};
    std::vector<S> data;
    Block() = default;
    Block(index_t r, index_t c, index_t tk) : rows(r), cols(c), t_k(tk) {
        if (r < 0 || c < 0 || tk < 1) throw Error(DIMENSION, "BlockMatrix: invalid shape");
        offsets.assign(1, 0);
        for (index_t b = 0; b < block_count(); ++b) offsets.push_back(offsets.back() + rows * block_width(b));
        data.assign(static_cast<std::size_t>(offsets.back()), zero<S>());
    }
    index_t block_count() const { return cols == 0 ? 0 : (cols + t_k - 1) / t_k; }
    index_t block_width(index_t b) const { return std::min(t_k, cols - b * t_k); }
    S* block(index_t b) { return data.data() + offsets[b]; }
    const S* block(index_t b) const { return data.data() + offsets[b]; }
    void set_zero() { std::fill(data.begin(), data.end(), zero<S>()); }
};

// to_block_layout / from_block_layout (tiled_matrix.hpp:151-175); the dense
// operand is column-major (Eigen default) with leading dimension ld.
template <class S>
Block<S> to_block_layout(const S* m, index_t rows, index_t cols, index_t ld, index_t t_k) {
    Block<S> out(rows, cols, t_k);
    for (index_t b = 0; b < out.block_count(); ++b) {
        const index_t c0 = b * t_k, w = out.block_width(b);
        S* dst = out.block(b);
        for (index_t r = 0; r < rows; ++r)
            for (index_t c = 0; c < w; ++c) dst[r * w + c] = m[(c0 + c) * ld + r];
    }
    return out;
}
template <class S>
void from_block_layout(const Block<S>& m, S* out, index_t ld) {
    for (index_t b = 0; b < m.block_count(); ++b) {
        const index_t c0 = b * m.t_k, w = m.block_width(b);
        const S* src = m.block(b);
        for (index_t r = 0; r < m.rows; ++r)
            for (index_t c = 0; c < w; ++c) out[(c0 + c) * ld + r] = src[r * w + c];
    }
}

// maspmm (tiled_matrix.hpp:184-210): C += A B; column blocks outer, row blocks
// in parallel, segments ascending column, entries ascending row.
template <class S>
void maspmm(const Tiled<S>& a, const Block<S>& b, Block<S>& c) {
    if (b.rows != a.n_cols || c.rows != a.n_rows || c.cols != b.cols)
        throw Error(DIMENSION, "maspmm: shape mismatch");
    if (b.t_k != a.t_k || c.t_k != a.t_k) throw Error(DIMENSION, "maspmm: dense block width does not match the tiling");
    if (b.cols == 0) return;
    const index_t nrb = a.row_blocks();
    for (index_t blk = 0; blk < b.block_count(); ++blk) {
        const index_t width = b.block_width(blk);
        const S* bdata = b.block(blk);
        S* cdata = c.block(blk);
#pragma omp parallel for schedule(static)
        for (index_t ib = 0; ib < nrb; ++ib) {
            for (index_t jj = a.act_colseg[ib]; jj < a.act_colseg[ib + 1]; ++jj) {
                const S* bseg = bdata + a.col_idx[jj] * width;
                for (index_t ii = a.colseg_ptr[jj]; ii < a.colseg_ptr[jj + 1]; ++ii) {
                    S* cseg = cdata + a.row_idx[ii] * width;
                    const S v = a.values[ii];
                    for (index_t t = 0; t < width; ++t) mac(cseg[t], v, bseg[t]);
                }
            }
        }
    }
}

// naive_spmm / csr_spmv (csr_matrix.hpp:122-147); column-major dense.
template <class S>
void naive_spmm(const Csr<S>& a, const S* b, index_t k, index_t ldb, S* c, index_t ldc) {
    for (index_t j = 0; j < k; ++j)
        for (index_t r = 0; r < a.n_rows; ++r) c[j * ldc + r] = zero<S>();
    for (index_t r = 0; r < a.n_rows; ++r)
        for (index_t kk = a.row_ptr[r]; kk < a.row_ptr[r + 1]; ++kk)
            for (index_t j = 0; j < k; ++j) mac(c[j * ldc + r], a.values[kk], b[j * ldb + a.col_idx[kk]]);
}

// ----------------------------------------------------------------- filter ---
// chebyshev_step_coeffs / lanczos_damping / jackson_damping / build_filter
// (proj/src/cheb_filter.cpp:21-94).
std::vector<double> step_coeffs(double alpha, double beta, int k) {
    if (!(0.0 <= beta && beta < alpha && alpha <= pi))
        throw Error(CONFIG, "chebyshev_step_coeffs: need 0 <= beta < alpha <= pi");
    if (k < 0) throw Error(CONFIG, "chebyshev_step_coeffs: negative degree");
    std::vector<double> c(static_cast<std::size_t>(k) + 1);
    c[0] = (alpha - beta) / pi;
    const bool a_pi = alpha == pi, b_pi = beta == pi;
    for (int j = 1; j <= k; ++j) {
        const double sa = a_pi ? 0.0 : std::sin(j * alpha);
        const double sb = b_pi ? 0.0 : std::sin(j * beta);
        c[j] = (2.0 / pi) * (sa - sb) / j;
    }
    return c;
}
std::vector<double> lanczos_damping(int k, double m) {
    if (k < 1) throw Error(CONFIG, "lanczos_damping: degree must be >= 1");
    if (m < 0.0) throw Error(CONFIG, "lanczos_damping: exponent must be >= 0");
    std::vector<double> d(static_cast<std::size_t>(k) + 1);
    d[0] = 1.0;
    for (int j = 1; j <= k; ++j) {
        const double u = j * pi / (k + 1);
        d[j] = std::pow(std::sin(u) / u, m);
    }
    return d;
}
std::vector<double> jackson_damping(int k) {
    if (k < 1) throw Error(CONFIG, "jackson_damping: degree must be >= 1");
    std::vector<double> d(static_cast<std::size_t>(k) + 1);
    d[0] = 1.0;
    const double h = pi / (k + 2);
    for (int j = 1; j <= k; ++j)
        d[j] = ((k + 2 - j) * std::sin(h) * std::cos(j * h) + std::cos(h) * std::sin(j * h)) / ((k + 2) * std::sin(h));
    return d;
}

}  // namespace orc

// ============================================================================
// C ABI for the Python test harness (ctypes). Dense operands column-major.
// ============================================================================
using namespace orc;

extern "C" {

struct orc_filter {  // ChebFilter (proj/include/adapoly/cheb_filter.hpp:41-66) minus coeffs
    double interval_a, interval_b, alpha, beta;
    int k_max;
    double m, l1, l2, lambda_min, lambda_max;
    int active_degree;
};

const char* orc_last_error(void) { return g_last_error.c_str(); }

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// --- Philox -----------------------------------------------------------------
void orc_philox_block(std::uint64_t seed, std::uint64_t stream, std::uint64_t counter, std::uint32_t* out) {
    Philox(seed, stream).block(counter, out);
}
// Raw Philox4x32-10 round function on an arbitrary 128-bit counter and 64-bit
// key (Random123 convention) -- used only for the published KAT vectors.
void orc_philox_raw(const std::uint32_t* ctr, const std::uint32_t* key, std::uint32_t* out) {
    std::uint64_t counter = ctr[0] | (std::uint64_t(ctr[1]) << 32);
    std::uint64_t stream = ctr[2] | (std::uint64_t(ctr[3]) << 32);
    std::uint64_t seed = key[0] | (std::uint64_t(key[1]) << 32);
    Philox(seed, stream).block(counter, out);
}
// fill_gaussian / fill_rademacher (philox.hpp:92-109): index c*n + r.
void orc_fill_gaussian(double* out, std::int64_t n, std::int64_t q, std::uint64_t seed, std::uint64_t stream) {
    const Philox rng(seed, stream);
#pragma omp parallel for schedule(static)
    for (index_t c = 0; c < q; ++c)
        for (index_t r = 0; r < n; ++r) out[c * n + r] = rng.gaussian(static_cast<std::uint64_t>(c * n + r));
}
void orc_fill_rademacher(double* out, std::int64_t n, std::int64_t q, std::uint64_t seed, std::uint64_t stream) {
    const Philox rng(seed, stream);
#pragma omp parallel for schedule(static)
    for (index_t c = 0; c < q; ++c)
        for (index_t r = 0; r < n; ++r) out[c * n + r] = rng.rademacher(static_cast<std::uint64_t>(c * n + r));
}
double orc_gaussian(std::uint64_t seed, std::uint64_t stream, std::uint64_t i) { return Philox(seed, stream).gaussian(i); }
void orc_gaussian_range(std::uint64_t seed, std::uint64_t stream, std::uint64_t first, std::int64_t count, double* out) {
    const Philox rng(seed, stream);
    for (index_t i = 0; i < count; ++i) out[i] = rng.gaussian(first + static_cast<std::uint64_t>(i));
}
void orc_uniform_range(std::uint64_t seed, std::uint64_t stream, std::uint64_t first, std::int64_t count, double* out) {
    const Philox rng(seed, stream);
#pragma omp parallel for schedule(static)
    for (index_t i = 0; i < count; ++i) out[i] = rng.uniform(first + static_cast<std::uint64_t>(i));
}

// --- std::mt19937_64 draws (libstdc++), to regenerate the reference tests'
// matrices bit for bit (proj/tests/support/test_matrices.hpp:25-65).
void* orc_mt_create(std::uint64_t seed) { return new std::mt19937_64(seed); }
void orc_mt_destroy(void* h) { delete static_cast<std::mt19937_64*>(h); }
std::uint64_t orc_mt_next(void* h) { return (*static_cast<std::mt19937_64*>(h))(); }
double orc_mt_uniform(void* h, double lo, double hi) {
    std::uniform_real_distribution<double> u(lo, hi);
    return u(*static_cast<std::mt19937_64*>(h));
}
std::int64_t orc_mt_uniform_int(void* h, std::int64_t lo, std::int64_t hi) {
    std::uniform_int_distribution<std::int64_t> u(lo, hi);
    return u(*static_cast<std::mt19937_64*>(h));
}
int orc_mt_bernoulli(void* h, double p) {
    std::bernoulli_distribution b(p);
    return b(*static_cast<std::mt19937_64*>(h)) ? 1 : 0;
}

// --- CSR handles ---------------------------------------------------------------
struct orc_csr {
    Csr<double> m;
};
struct orc_zcsr {
    Csr<cplx> m;
};

static void csr_from_triplet_vec(orc_csr* h, index_t rows, index_t cols, std::vector<Triplet<double>> t) {
    h->m = from_triplets<double>(rows, cols, std::move(t));
}

int orc_csr_from_triplets(std::int64_t rows, std::int64_t cols, std::int64_t nt, const std::int64_t* r,
                          const std::int64_t* c, const double* v, orc_csr** out) {
    return guarded([&] {
        std::vector<Triplet<double>> t(static_cast<std::size_t>(nt));
        for (index_t i = 0; i < nt; ++i) t[i] = {r[i], c[i], v[i]};
        auto* h = new orc_csr;
        try {
            csr_from_triplet_vec(h, rows, cols, std::move(t));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
// random_csr / random_symmetric (test_matrices.hpp:38-65): mt19937_64 with
// uniform_real_distribution(-1,1) and bernoulli_distribution(density), same
// draw order.
orc_csr* orc_random_csr(std::int64_t rows, std::int64_t cols, double density, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> value(-1.0, 1.0);
    std::bernoulli_distribution keep(density);
    std::vector<Triplet<double>> t;
    for (index_t r = 0; r < rows; ++r)
        for (index_t c = 0; c < cols; ++c)
            if (keep(rng)) t.push_back({r, c, value(rng)});
    auto* h = new orc_csr;
    csr_from_triplet_vec(h, rows, cols, std::move(t));
    return h;
}
orc_csr* orc_random_symmetric(std::int64_t n, double density, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> value(-1.0, 1.0);
    std::bernoulli_distribution keep(density);
    std::vector<Triplet<double>> t;
    for (index_t r = 0; r < n; ++r)
        for (index_t c = r; c < n; ++c) {
            if (!keep(rng)) continue;
            const double v = value(rng);
            t.push_back({r, c, v});
            if (c != r) t.push_back({c, r, v});
        }
    auto* h = new orc_csr;
    csr_from_triplet_vec(h, n, n, std::move(t));
    return h;
}
// Wrap an existing CSR (already sorted, no duplicates; e.g. a generator output).
orc_csr* orc_csr_wrap(std::int64_t rows, std::int64_t cols, const std::int64_t* rp, const std::int64_t* ci,
                      const double* v) {
    auto* h = new orc_csr;
    h->m.n_rows = rows;
    h->m.n_cols = cols;
    h->m.row_ptr.assign(rp, rp + rows + 1);
    h->m.col_idx.assign(ci, ci + rp[rows]);
    h->m.values.assign(v, v + rp[rows]);
    return h;
}
orc_csr* orc_csr_wrap32(std::int64_t rows, std::int64_t cols, const std::int64_t* rp, const std::int32_t* ci,
                        const double* v) {
    auto* h = new orc_csr;
    h->m.n_rows = rows;
    h->m.n_cols = cols;
    h->m.row_ptr.assign(rp, rp + rows + 1);
    h->m.col_idx.assign(ci, ci + rp[rows]);
    h->m.values.assign(v, v + rp[rows]);
    return h;
}
void orc_csr_destroy(orc_csr* h) { delete h; }
void orc_csr_dims(const orc_csr* h, std::int64_t* rows, std::int64_t* cols, std::int64_t* nnz) {
    *rows = h->m.n_rows;
    *cols = h->m.n_cols;
    *nnz = h->m.nnz();
}
void orc_csr_export(const orc_csr* h, std::int64_t* rp, std::int64_t* ci, double* v) {
    std::copy(h->m.row_ptr.begin(), h->m.row_ptr.end(), rp);
    std::copy(h->m.col_idx.begin(), h->m.col_idx.end(), ci);
    std::copy(h->m.values.begin(), h->m.values.end(), v);
}

orc_zcsr* orc_zcsr_wrap(std::int64_t rows, std::int64_t cols, const std::int64_t* rp, const std::int64_t* ci,
                        const double* v_interleaved) {
    auto* h = new orc_zcsr;
    h->m.n_rows = rows;
    h->m.n_cols = cols;
    h->m.row_ptr.assign(rp, rp + rows + 1);
    h->m.col_idx.assign(ci, ci + rp[rows]);
    h->m.values.resize(static_cast<std::size_t>(rp[rows]));
    for (index_t k = 0; k < rp[rows]; ++k) h->m.values[k] = {v_interleaved[2 * k], v_interleaved[2 * k + 1]};
    return h;
}
void orc_zcsr_destroy(orc_zcsr* h) { delete h; }

// --- tiled handles -------------------------------------------------------------
struct orc_tiled {
    Tiled<double> t;
};
struct orc_ztiled {
    Tiled<cplx> t;
};
int orc_tiled_create(const orc_csr* a, std::int64_t ti, std::int64_t tk, orc_tiled** out) {
    return guarded([&] {
        auto* h = new orc_tiled;
        try {
            h->t = csr_to_tiled(a->m, ti, tk);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
int orc_ztiled_create(const orc_zcsr* a, std::int64_t ti, std::int64_t tk, orc_ztiled** out) {
    return guarded([&] {
        auto* h = new orc_ztiled;
        try {
            h->t = csr_to_tiled(a->m, ti, tk);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
void orc_tiled_destroy(orc_tiled* h) { delete h; }
void orc_ztiled_destroy(orc_ztiled* h) { delete h; }
void orc_tiled_sizes(const orc_tiled* h, std::int64_t* n_segs, std::int64_t* n_blocks, std::int64_t* nnz) {
    *n_segs = static_cast<std::int64_t>(h->t.col_idx.size());
    *n_blocks = h->t.row_blocks();
    *nnz = static_cast<std::int64_t>(h->t.values.size());
}
void orc_tiled_export(const orc_tiled* h, std::int64_t* act_colseg, std::int64_t* colseg_ptr, std::int64_t* col_idx,
                      std::int64_t* row_idx, double* values) {
    std::copy(h->t.act_colseg.begin(), h->t.act_colseg.end(), act_colseg);
    std::copy(h->t.colseg_ptr.begin(), h->t.colseg_ptr.end(), colseg_ptr);
    std::copy(h->t.col_idx.begin(), h->t.col_idx.end(), col_idx);
    std::copy(h->t.row_idx.begin(), h->t.row_idx.end(), row_idx);
    std::copy(h->t.values.begin(), h->t.values.end(), values);
}

// maspmm through the block layout: C (col-major, n_rows x k) += A B.
int orc_maspmm(const orc_tiled* a, const double* b, std::int64_t k, double* c) {
    return guarded([&] {
        const Tiled<double>& t = a->t;
        Block<double> bb = to_block_layout(b, t.n_cols, k, t.n_cols, t.t_k);
        Block<double> cc = to_block_layout(c, t.n_rows, k, t.n_rows, t.t_k);
        maspmm(t, bb, cc);
        from_block_layout(cc, c, t.n_rows);
    });
}
// Shape-checked maspmm on explicit block shapes (for the DimensionError tests).
int orc_maspmm_shapes(const orc_tiled* a, std::int64_t b_rows, std::int64_t b_cols, std::int64_t b_tk,
                      std::int64_t c_rows, std::int64_t c_cols, std::int64_t c_tk) {
    return guarded([&] {
        Block<double> bb(b_rows, b_cols, b_tk), cc(c_rows, c_cols, c_tk);
        maspmm(a->t, bb, cc);
    });
}
int orc_naive_spmm(const orc_csr* a, const double* b, std::int64_t k, double* c) {
    return guarded([&] {
        naive_spmm(a->m, b, k, a->m.n_cols, c, a->m.n_rows);
    });
}
int orc_csr_spmv(const orc_csr* a, const double* x, double* y) {  // csr_matrix.hpp:122-134
    return guarded([&] {
        for (index_t r = 0; r < a->m.n_rows; ++r) {
            double acc = 0.0;
            for (index_t k = a->m.row_ptr[r]; k < a->m.row_ptr[r + 1]; ++k) acc += a->m.values[k] * x[a->m.col_idx[k]];
            y[r] = acc;
        }
    });
}

// --- filter construction ---------------------------------------------------------
int orc_step_coeffs(double alpha, double beta, int k, double* out) {
    return guarded([&] {
        auto c = step_coeffs(alpha, beta, k);
        std::copy(c.begin(), c.end(), out);
    });
}
int orc_lanczos_damping(int k, double m, double* out) {
    return guarded([&] {
        auto d = lanczos_damping(k, m);
        std::copy(d.begin(), d.end(), out);
    });
}
int orc_jackson_damping(int k, double* out) {
    return guarded([&] {
        auto d = jackson_damping(k);
        std::copy(d.begin(), d.end(), out);
    });
}
static double map_clamped(const orc_filter* f, double x, bool* clamped) {  // cheb_filter.hpp:55-62
    const double t = f->l1 * x + f->l2;
    if (t < -1.0 || t > 1.0) {
        if (clamped) *clamped = true;
        return t < -1.0 ? -1.0 : 1.0;
    }
    return t;
}
// build_filter (cheb_filter.cpp:63-94); damping 0 = lanczos, 1 = jackson.
int orc_build_filter(double a, double b, double lmin, double lmax, int k, double m, int damping, orc_filter* f,
                     double* coeffs) {
    return guarded([&] {
        if (!std::isfinite(lmin) || !std::isfinite(lmax) || !(lmin < lmax))
            throw Error(CONFIG, "build_filter: invalid spectrum bounds");
        if (!(lmin <= a && a < b && b <= lmax))
            throw Error(CONFIG, "build_filter: target interval must lie inside the spectrum bounds");
        if (k < 1) throw Error(CONFIG, "build_filter: degree must be >= 1");
        if (m < 0.0) throw Error(CONFIG, "build_filter: damping exponent must be >= 0");
        f->interval_a = a;
        f->interval_b = b;
        f->k_max = k;
        f->m = m;
        f->lambda_min = lmin;
        f->lambda_max = lmax;
        const double span = lmax - lmin;
        f->l1 = 2.0 / span;
        f->l2 = -(lmax + lmin) / span;
        f->alpha = std::acos(map_clamped(f, a, nullptr));
        f->beta = std::acos(map_clamped(f, b, nullptr));
        if (!(f->alpha > f->beta)) throw Error(CONFIG, "build_filter: interval collapses under the spectral map");
        const auto c = step_coeffs(f->alpha, f->beta, k);
        const auto d = damping == 0 ? lanczos_damping(k, m) : jackson_damping(k);
        for (std::size_t j = 0; j < c.size(); ++j) coeffs[j] = c[j] * d[j];
        f->active_degree = k;
    });
}
// eval_filter_scalar (cheb_filter.cpp:96-111).
double orc_eval_filter_scalar(const orc_filter* f, const double* coeffs, double x, int degree) {
    const double t = map_clamped(f, x, nullptr);
    double acc = coeffs[0];
    if (degree >= 1) {
        double t_prev = 1.0, t_cur = t;
        acc += coeffs[1] * t_cur;
        for (int j = 2; j <= degree; ++j) {
            const double t_next = 2.0 * t * t_cur - t_prev;
            acc += coeffs[j] * t_next;
            t_prev = t_cur;
            t_cur = t_next;
        }
    }
    return acc;
}
// Vector form with clamp count (cheb_filter.cpp:113-127).
int orc_eval_filter_vector(const orc_filter* f, const double* coeffs, const double* x, std::int64_t n, int degree,
                           double* out, std::int64_t* clamped) {
    return guarded([&] {
        if (degree < 0 || degree > f->k_max) throw Error(CONFIG, "eval_filter_scalar: degree out of range");
        index_t nc = 0;
        for (index_t i = 0; i < n; ++i) {
            bool c = false;
            map_clamped(f, x[i], &c);
            nc += c ? 1 : 0;
            out[i] = orc_eval_filter_scalar(f, coeffs, x[i], degree);
        }
        if (clamped) *clamped += nc;
    });
}

// initial_degree / adaptive_degree (cheb_filter.cpp:181-219).
int orc_initial_degree(double alpha, double beta, double c, int* out) {
    return guarded([&] {
        const double width = alpha - beta;
        if (!(width > 0.0)) throw Error(CONFIG, "initial_degree: need alpha > beta");
        if (!(c > width)) throw Error(CONFIG, "initial_degree: constant must exceed alpha - beta");
        const int k1 = static_cast<int>(std::ceil(c / width)) - 1;
        *out = std::max(k1, 1);
    });
}
int orc_adaptive_degree(const orc_filter* f, const double* coeffs, const double* ritz, std::int64_t p,
                        std::int64_t e_i, double tau_a, int* out) {
    return guarded([&] {
        if (p < 1) throw Error(CONFIG, "adaptive_degree: empty Ritz set");
        if (e_i < 1 || e_i > p) throw Error(CONFIG, "adaptive_degree: in-interval count out of range");
        if (!(tau_a > 0.0)) throw Error(CONFIG, "adaptive_degree: threshold must be positive");
        const int floor_degree = std::min(3, f->k_max);
        std::vector<double> t(p), h_prev(p, 1.0), h_cur(p), gamma(p, coeffs[0]), mags(p), h_next(p);
        for (index_t i = 0; i < p; ++i) t[i] = map_clamped(f, ritz[i], nullptr);
        h_cur = t;
        for (int j = 1; j <= f->k_max; ++j) {
            for (index_t i = 0; i < p; ++i) gamma[i] += coeffs[j] * h_cur[i];
            for (index_t i = 0; i < p; ++i) mags[i] = std::abs(gamma[i]);
            std::sort(mags.begin(), mags.end(), std::greater<double>());
            const double denom = mags[e_i - 1], num = mags[p - 1];
            if (denom > 0.0 && num / denom < tau_a) {
                *out = std::min(std::max(j, floor_degree), f->k_max);
                return;
            }
            for (index_t i = 0; i < p; ++i) h_next[i] = 2.0 * t[i] * h_cur[i] - h_prev[i];
            h_prev = h_cur;
            h_cur = h_next;
        }
        *out = f->k_max;
    });
}

}  // extern "C"

// ---------------------------------------------------------------- clenshaw ---
// clenshaw_apply (proj/src/cheb_filter.cpp:129-179), restated on the block
// layout with the exact expression order of the Eigen array updates.
namespace orc {
template <class S>
void clenshaw_apply(const double* coeffs, int k_max, double l1, double l2, const Tiled<S>& a, const S* x,
                    index_t n, index_t q, int degree, S* out, std::int64_t* spmv_count) {
    if (degree < 0 || degree > k_max) throw Error(CONFIG, "clenshaw_apply: degree out of range");
    if (n != a.n_cols) throw Error(DIMENSION, "clenshaw_apply: operand row count does not match A");
    if (q == 0) return;
    int deg = degree;
    while (deg > 0 && coeffs[deg] == 0.0) --deg;
    if (spmv_count) *spmv_count += static_cast<std::int64_t>(deg) * q;
    const index_t total = n * q;
    if (deg == 0) {
        for (index_t i = 0; i < total; ++i) out[i] = coeffs[0] * x[i];
        return;
    }
    Block<S> y = to_block_layout(x, n, q, n, a.t_k);
    Block<S> aw(a.n_rows, q, a.t_k);
    if (deg == 1) {
        maspmm(a, y, aw);
        std::vector<S> o(static_cast<std::size_t>(total));
        from_block_layout(aw, o.data(), n);
        // f.coeffs[0] * x + f.coeffs[1] * (f.l1 * out + f.l2 * x)
        for (index_t i = 0; i < total; ++i) out[i] = coeffs[0] * x[i] + coeffs[1] * (l1 * o[i] + l2 * x[i]);
        return;
    }
    Block<S> w(a.n_rows, q, a.t_k), v(a.n_rows, q, a.t_k);
    const std::size_t sz = y.data.size();
    const double cd = coeffs[deg];
    for (std::size_t i = 0; i < sz; ++i) w.data[i] = cd * y.data[i];
    maspmm(a, w, aw);
    const double two_l1 = 2.0 * l1, two_l2 = 2.0 * l2;
    const double first = 2.0 * l2 + coeffs[deg - 1] / coeffs[deg];
    for (std::size_t i = 0; i < sz; ++i) v.data[i] = two_l1 * aw.data[i] + first * w.data[i];
    std::swap(v, w);
    for (int j = deg - 2; j >= 1; --j) {
        aw.set_zero();
        maspmm(a, w, aw);
        const double cj = coeffs[j];
        S* vd = v.data.data();
        const S* ad = aw.data.data();
        const S* wd = w.data.data();
        const S* yd = y.data.data();
        // Eigen coefficient-wise expressions are single-threaded in the
        // reference (OpenMP only reaches maspmm), so this loop is too.
        for (std::size_t i = 0; i < sz; ++i) vd[i] = two_l1 * ad[i] + two_l2 * wd[i] - vd[i] + cj * yd[i];
        std::swap(v, w);
    }
    aw.set_zero();
    maspmm(a, w, aw);
    const double c0 = coeffs[0];
    for (std::size_t i = 0; i < sz; ++i) v.data[i] = l1 * aw.data[i] + l2 * w.data[i] - v.data[i] + c0 * y.data[i];
    from_block_layout(v, out, n);
}
}  // namespace orc

extern "C" {

int orc_clenshaw_apply(const double* coeffs, int k_max, double l1, double l2, const orc_tiled* a, const double* x,
                       std::int64_t n, std::int64_t q, int degree, double* out, std::int64_t* spmv_count) {
    return guarded([&] { clenshaw_apply<double>(coeffs, k_max, l1, l2, a->t, x, n, q, degree, out, spmv_count); });
}
// Complex: x / out are interleaved (re, im) column-major n x q.
int orc_zclenshaw_apply(const double* coeffs, int k_max, double l1, double l2, const orc_ztiled* a, const double* x,
                        std::int64_t n, std::int64_t q, int degree, double* out, std::int64_t* spmv_count) {
    return guarded([&] {
        clenshaw_apply<cplx>(coeffs, k_max, l1, l2, a->t, reinterpret_cast<const cplx*>(x), n, q, degree,
                             reinterpret_cast<cplx*>(out), spmv_count);
    });
}

// estimate_eigcount (proj/src/solver.cpp:108-117): Rademacher probes from
// stream 2, filter at k_max, mean of v^T w.
int orc_estimate_eigcount(const double* coeffs, int k_max, double l1, double l2, const orc_tiled* a,
                          std::int64_t probes, std::uint64_t seed, double* out, std::int64_t* spmv_count) {
    return guarded([&] {
        if (probes < 1) throw Error(CONFIG, "estimate_eigcount: need at least one probe");
        const index_t n = a->t.n_rows;
        std::vector<double> v(static_cast<std::size_t>(n * probes)), w(v.size());
        orc_fill_rademacher(v.data(), n, probes, seed, 2);
        clenshaw_apply<double>(coeffs, k_max, l1, l2, a->t, v.data(), n, probes, k_max, w.data(), spmv_count);
        double acc = 0.0;
        for (index_t c = 0; c < probes; ++c) {
            // Eigen dot(): a reduction whose association order is Eigen's; the
            // estimate is statistical and compared with tolerance only.
            double d = 0.0;
            for (index_t r = 0; r < n; ++r) d += v[c * n + r] * w[c * n + r];
            acc += d;
        }
        *out = acc / static_cast<double>(probes);
    });
}

// CPU baseline timing: `steps` middle Clenshaw steps (maspmm + array update,
// cheb_filter.cpp:167-173) on block-layout operands; returns seconds, timed
// with steady_clock like bench-spmm (proj/src/cli.cpp:259-279).
int orc_bench_clenshaw_steps(const orc_tiled* a, std::int64_t q, int steps, double* seconds, double* checksum) {
    return guarded([&] {
        const Tiled<double>& t = a->t;
        const index_t n = t.n_rows;
        Block<double> y(n, q, t.t_k), w(n, q, t.t_k), v(n, q, t.t_k), aw(n, q, t.t_k);
        const Philox rng(7, 7);
        const std::size_t sz = y.data.size();
#pragma omp parallel for schedule(static)
        for (std::size_t i = 0; i < sz; ++i) {
            y.data[i] = rng.uniform(i) - 0.5;
            w.data[i] = 0.5 * y.data[i];
            v.data[i] = 0.25 * y.data[i];
        }
        const double two_l1 = 0.25, two_l2 = -0.5, cj = 0.01;
        const auto t0 = std::chrono::steady_clock::now();
        for (int s = 0; s < steps; ++s) {
            aw.set_zero();
            maspmm(t, w, aw);
            double* vd = v.data.data();
            const double* ad = aw.data.data();
            const double* wd = w.data.data();
            const double* yd = y.data.data();
            for (std::size_t i = 0; i < sz; ++i) vd[i] = two_l1 * ad[i] + two_l2 * wd[i] - vd[i] + cj * yd[i];
            std::swap(v, w);
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        double cs = 0.0;
        for (std::size_t i = 0; i < sz; i += 97) cs += w.data[i];
        *checksum = cs;
    });
}

}  // extern "C"
