"""Pin the CPU oracle to the reference (CPU only, no GPU).

Every test here restates one of the reference's own known-answer / oracle
tests for the hot path (file:line cited) against oracle/oracle.cpp, using the
reference's own generators bit for bit (libstdc++ mt19937_64 + distributions,
proj/tests/support/test_matrices.hpp) and its three .mtx fixtures (converted
to tests/golden/fixture_*.npz by tests/golden/make_golden.py). Passing these
is what licenses the oracle as the parity checker for the CUDA path.
"""
import math

import numpy as np
import pytest

PI = math.pi


def rel_fro(got, want):
    d = np.linalg.norm(want)
    return np.linalg.norm(got - want) / d if d > 0 else np.linalg.norm(got - want)


def unit_bounds():
    return (-1.0, 1.0)


def load_fixture(orc, golden_dir, name):
    z = np.load(f"{golden_dir}/fixture_{name}.npz")
    return orc.Csr(int(z["n_rows"]), int(z["n_cols"]), z["row_ptr"], z["col_idx"], z["values"])


# ------------------------------------------------------------- Philox KATs ---
@pytest.mark.parametrize("ctr,key,want", [
    # Published Philox4x32-10 known-answer vectors (Salmon et al. SC'11, Random123 kat_vectors).
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
])
def test_philox_known_answers(orc, ctr, key, want):
    assert list(orc.philox_raw(ctr, key)) == want


def test_philox_fill_addressing(orc):
    # fill_gaussian index = c*n + r (philox.hpp:96-98); draw i uses block i/4, Box-Muller pair (i%4)/2.
    n, q = 7, 3
    g = orc.fill_gaussian(n, q, 5, 1)
    flat = orc.gaussian_range(5, 1, 0, n * q)
    assert np.array_equal(g.ravel(order="F"), flat)
    b = orc.philox_block(5, 1, 0)
    u1, u2 = (b[0] + 0.5) * 2.0 ** -32, (b[1] + 0.5) * 2.0 ** -32
    r = math.sqrt(-2.0 * math.log(u1))
    assert flat[0] == r * math.cos(2.0 * PI * u2)
    assert flat[1] == r * math.sin(2.0 * PI * u2)
    rad = orc.fill_rademacher(n, q, 5, 2)
    assert set(np.unique(rad)) <= {-1.0, 1.0}
    words = np.concatenate([orc.philox_block(5, 2, i) for i in range(6)])
    assert np.array_equal(rad.ravel(order="F"), np.where(words[: n * q] >> 31, 1.0, -1.0))


# ------------------------------------------------- coefficients and damping ---
def test_step_coeffs_full_interval(orc):  # test_cheb_filter.cpp:48-52
    c = orc.chebyshev_step_coeffs(PI, 0.0, 12)
    assert c[0] == 1.0 and np.all(c[1:] == 0.0)


def test_step_coeffs_symmetric_kills_odd(orc):  # :54-58
    c = orc.chebyshev_step_coeffs(PI - 0.7, 0.7, 15)
    assert np.all(np.abs(c[1::2]) <= 5e-16)


def test_step_coeffs_plugin(orc):  # :60-68
    alpha, beta = math.acos(0.1), math.acos(0.6)
    c = orc.chebyshev_step_coeffs(alpha, beta, 3)
    want1 = (2.0 / PI) * (math.sqrt(1.0 - 0.01) - 0.8)
    assert c[1] == pytest.approx(want1, rel=1e-15)
    assert c[0] == pytest.approx((alpha - beta) / PI, rel=1e-15)


def test_step_coeffs_long_double(orc):  # :70-86
    alpha, beta = 2.2143, 0.4377
    c = orc.chebyshev_step_coeffs(alpha, beta, 40)
    scale = np.abs(c).max()
    ld = np.longdouble
    for j in range(1, 41):
        want = (ld(2) / ld(PI)) * (np.sin(ld(j) * ld(alpha)) - np.sin(ld(j) * ld(beta))) / ld(j)
        assert abs(c[j] - float(want)) <= 1e-15 * scale
    with pytest.raises(orc.ConfigError):
        orc.chebyshev_step_coeffs(0.4, 0.5, 3)


def test_lanczos_damping(orc):  # :88-104
    assert np.all(orc.lanczos_damping(9, 0.0) == 1.0)
    d31 = orc.lanczos_damping(3, 1.0)
    assert d31[0] == 1.0 and d31[2] == pytest.approx(2.0 / PI, rel=1e-15)
    d = orc.lanczos_damping(20, 0.5)
    assert np.all(d[1:] > 0) and np.all(d[1:] <= 1.0) and np.all(d[1:] < d[:-1])
    with pytest.raises(orc.ConfigError):
        orc.lanczos_damping(10, -0.5)
    with pytest.raises(orc.ConfigError):
        orc.lanczos_damping(0, 1.0)


def test_jackson_damping(orc):  # :106-114
    d = orc.jackson_damping(4)
    h = PI / 6.0
    want1 = (5.0 * math.sin(h) * math.cos(h) + math.cos(h) * math.sin(h)) / (6.0 * math.sin(h))
    assert d[0] == 1.0 and d[1] == pytest.approx(want1, rel=1e-14)
    assert np.all(d[1:] < d[:-1])


def test_build_filter_invariants(orc):  # :116-131
    f = orc.build_filter(0.1, 0.6, unit_bounds(), 30, 0.5)
    assert f.alpha == pytest.approx(math.acos(0.1), rel=1e-15)
    assert f.beta == pytest.approx(math.acos(0.6), rel=1e-15)
    assert f.alpha > f.beta >= 0.0 and f.alpha <= PI
    assert f.coeffs[0] == pytest.approx((f.alpha - f.beta) / PI, rel=1e-15)
    assert f.active_degree == 30 and f.k_max == 30
    assert f.map(0.1) == pytest.approx(0.1)
    for args in [(-2.0, 0.5, unit_bounds(), 10, 0.5), (0.5, 0.1, unit_bounds(), 10, 0.5),
                 (0.1, 0.6, unit_bounds(), 0, 0.5)]:
        with pytest.raises(orc.ConfigError):
            orc.build_filter(*args)


def test_build_filter_full_interval_is_one(orc):  # :133-137
    f = orc.build_filter(-1.0, 1.0, unit_bounds(), 25, 0.5)
    for x in (-1.0, -0.33, 0.0, 0.5, 1.0):
        assert orc.eval_filter_scalar(f, x, 25) == 1.0


def test_m0_equals_undamped_series(orc):  # :139-148
    f = orc.build_filter(0.1, 0.6, unit_bounds(), 40, 0.0)
    c = orc.chebyshev_step_coeffs(f.alpha, f.beta, 40)
    x = -0.95
    while x <= 0.95:
        th = math.acos(x)
        direct = sum(c[j] * math.cos(j * th) for j in range(41))
        assert orc.eval_filter_scalar(f, x, 40) == pytest.approx(direct, rel=1e-12)
        x += 0.1


def test_midpoint_approaches_one(orc):  # :150-161
    f = orc.build_filter(0.1, 0.6, unit_bounds(), 200, 0.0)
    val = orc.eval_filter_scalar(f, 0.35, 200)
    assert abs(val - 1.0) <= 0.05
    c = orc.chebyshev_step_coeffs(f.alpha, f.beta, 200)
    th = math.acos(0.35)
    assert val == pytest.approx(sum(c[j] * math.cos(j * th) for j in range(201)), rel=1e-12)


def test_degree1_affine(orc):  # :163-169
    f = orc.build_filter(-0.2, 0.9, (-2.0, 3.0), 10, 0.7)
    for x in (-1.5, 0.0, 0.4, 2.5):
        assert orc.eval_filter_scalar(f, x, 1) == pytest.approx(f.coeffs[0] + f.coeffs[1] * f.map(x), rel=1e-15)


def test_clamp_counting(orc):  # :171-180
    f = orc.build_filter(0.1, 0.6, unit_bounds(), 30, 0.5)
    vals, clamped = orc.eval_filter_scalar(f, np.array([-1.5, 0.3, 2.0]), 30)
    assert clamped == 2
    assert vals[0] == orc.eval_filter_scalar(f, -1.0, 30)
    assert vals[2] == orc.eval_filter_scalar(f, 1.0, 30)


def test_even_filter_symmetry(orc):  # :182-187
    f = orc.build_filter(-0.4, 0.4, unit_bounds(), 60, 0.5)
    for i in range(21):
        x = 0.05 * i
        assert abs(orc.eval_filter_scalar(f, x, 60) - orc.eval_filter_scalar(f, -x, 60)) <= 1e-13


# ----------------------------------------------------------- clenshaw_apply ---
def test_clenshaw_diagonal_factorizes(orc):  # :189-209
    rng = orc.MT19937_64(3)
    diag = [rng.uniform(-0.95, 0.95) for _ in range(40)]
    t = orc.Tiled(orc.make_diag(diag), 16, 4)
    f = orc.build_filter(-0.3, 0.5, unit_bounds(), 35, 0.5)
    x = orc.fill_gaussian(40, 3, 5, 1)
    for degree in (1, 2, 7, 35):
        got = orc.clenshaw_apply(f, t, x, degree)
        for i in range(40):
            rho = orc.eval_filter_scalar(f, diag[i], degree)
            want = rho * x[i]
            # doctest Approx(want).epsilon(1e-12).scale(1.0): |got-want| < 1e-12 (1 + max|.|)
            tol = 1e-12 * (1.0 + np.maximum(np.abs(got[i]), np.abs(want)))
            assert np.all(np.abs(got[i] - want) < tol)


def test_clenshaw_full_interval_returns_x_exactly(orc):  # :211-223
    a = orc.random_symmetric(30, 0.2, 9)
    t = orc.Tiled(a, 8, 4)
    f = orc.build_filter(-40.0, 40.0, (-40.0, 40.0), 20, 0.5)
    x = orc.fill_gaussian(30, 4, 2, 0)
    spmv = [0]
    got = orc.clenshaw_apply(f, t, x, 20, spmv)
    assert np.array_equal(got, x) and spmv[0] == 0


def test_clenshaw_equals_forward_oracle(orc):  # :225-240
    a = orc.random_symmetric(80, 0.1, 31)
    spec = np.linalg.eigvalsh(a.to_dense())
    f = orc.build_filter(spec[10], spec[50], (spec[0] - 0.1, spec[-1] + 0.1), 60, 0.5)
    t = orc.Tiled(a, 16, 8)
    x = orc.fill_gaussian(80, 6, 77, 3)
    for degree in (2, 3, 25, 60):
        assert rel_fro(orc.clenshaw_apply(f, t, x, degree), orc.forward_filter_apply(f, a.to_dense(), x, degree)) <= 1e-11


def test_clenshaw_trailing_zero_reduction(orc):  # :242-254
    a = orc.make_diag([0.1, -0.4, 0.7, 0.2])
    t = orc.Tiled(a, 2, 2)
    f = orc.build_filter(-0.5, 0.5, unit_bounds(), 5, 0.0)
    f.coeffs = np.array([0.3, 0.5, 0.2, 0.0, 0.0, 0.0])
    x = orc.fill_gaussian(4, 2, 1, 0)
    spmv = [0]
    got = orc.clenshaw_apply(f, t, x, 5, spmv)
    assert spmv[0] == 4
    assert rel_fro(got, orc.forward_filter_apply(f, a.to_dense(), x, 2)) <= 1e-14


def test_clenshaw_spmv_accounting(orc):  # :256-268
    a = orc.random_symmetric(24, 0.3, 12)
    t = orc.Tiled(a, 8, 4)
    f = orc.build_filter(-2.0, 5.0, (-30.0, 30.0), 12, 0.5)
    x = orc.fill_gaussian(24, 5, 8, 2)
    spmv = [0]
    orc.clenshaw_apply(f, t, x, 12, spmv)
    assert spmv[0] == 60
    orc.clenshaw_apply(f, t, x, 3, spmv)
    assert spmv[0] == 75
    with pytest.raises(orc.ConfigError):
        orc.clenshaw_apply(f, t, x, 13)
    with pytest.raises(orc.DimensionError):
        orc.clenshaw_apply(f, t, x[:20], 3)


def test_initial_degree(orc):  # :270-278
    assert orc.initial_degree(0.9, 0.4, 1.0) == 1
    assert orc.initial_degree(0.5, 0.3, 1.4) == 6
    assert orc.initial_degree(math.acos(0.1), math.acos(0.6), 1.4) == 2
    assert orc.initial_degree(1.0, 0.2, 0.81) == 1
    with pytest.raises(orc.ConfigError):
        orc.initial_degree(1.0, 0.5, 0.4)


def test_adaptive_degree_degenerate(orc):  # :280-291
    f = orc.build_filter(-0.2, 0.3, unit_bounds(), 25, 0.5)
    ritz = [-0.1, 0.0, 0.1, 0.25]
    assert orc.adaptive_degree(f, ritz, 4, 1e-3) == 25
    assert orc.adaptive_degree(f, [0.05] * 6, 2, 1e-3) == 25
    for e in (0, 5):
        with pytest.raises(orc.ConfigError):
            orc.adaptive_degree(f, ritz, e, 1e-3)


def test_adaptive_degree_floor(orc):  # :293-299
    f = orc.build_filter(-0.5, 0.5, unit_bounds(), 30, 0.5)
    assert orc.adaptive_degree(f, [0.0, 0.98], 1, 0.999) == 3


def test_adaptive_degree_exhaustive_scan(orc):  # :301-330
    a = orc.random_symmetric(50, 0.2, 41)
    spec = np.linalg.eigvalsh(a.to_dense())
    lo, hi = spec[20] - 1e-6, spec[32] + 1e-6
    f = orc.build_filter(lo, hi, (spec[0] - 0.05, spec[49] + 0.05), 80, 0.5)
    e = int(np.sum((spec >= lo) & (spec <= hi)))
    assert e == 13
    got = orc.adaptive_degree(f, spec, e, 1e-3)
    want = f.k_max
    for j in range(1, f.k_max + 1):
        mags = sorted((abs(orc.eval_filter_scalar(f, s, j)) for s in spec), reverse=True)
        if mags[-1] / mags[e - 1] < 1e-3:
            want = j
            break
    assert got == min(max(want, 3), f.k_max)


def test_adaptive_degree_monotone(orc):  # :332-344
    a = orc.random_symmetric(40, 0.25, 15)
    spec = np.linalg.eigvalsh(a.to_dense())
    f = orc.build_filter(spec[15] - 1e-8, spec[25] + 1e-8, (spec[0] - 0.05, spec[39] + 0.05), 120, 0.5)
    prev = 10 ** 9
    for tau in (1e-5, 1e-4, 1e-3, 1e-2, 1e-1):
        deg = orc.adaptive_degree(f, spec, 11, tau)
        assert deg <= prev
        prev = deg


# ---------------------------------------------------------- tiled + maspmm ---
def test_tiled_single_block_lists_sorted_distinct_columns(orc):  # test_sparse_core.cpp:164-180
    a = orc.random_csr(9, 9, 0.3, 3)
    ex = orc.Tiled(a, 100, 8).export()
    assert len(ex["act_colseg"]) == 2
    assert list(ex["col_idx"]) == sorted(set(a.col_idx.tolist()))


def test_tiled_tridiagonal_blocks(orc):  # :182-199
    r, c, v = [], [], []
    for i in range(4):
        r.append(i); c.append(i); v.append(2.0)
        if i > 0:
            r.append(i); c.append(i - 1); v.append(-1.0)
        if i < 3:
            r.append(i); c.append(i + 1); v.append(-1.0)
    ex = orc.Tiled(orc.Csr.from_triplets(4, 4, r, c, v), 2, 4).export()
    act, ci = ex["act_colseg"], ex["col_idx"]
    assert len(act) == 3
    assert list(ci[act[0]:act[1]]) == [0, 1, 2] and list(ci[act[1]:act[2]]) == [1, 2, 3]


def test_tiled_round_trip(orc):  # :201-219
    for ti in (1, 3, 64):
        a = orc.random_csr(37, 29, 0.2, 100 + ti)
        ex = orc.Tiled(a, ti, 8).export()
        trip = set()
        for jj in range(len(ex["col_idx"])):
            for ii in range(ex["colseg_ptr"][jj], ex["colseg_ptr"][jj + 1]):
                trip.add((int(ex["row_idx"][ii]), int(ex["col_idx"][jj]), float(ex["values"][ii])))
        rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr))
        assert trip == set(zip(rows.tolist(), a.col_idx.tolist(), a.values.tolist()))
        for ib in range(len(ex["act_colseg"]) - 1):
            for jj in range(ex["act_colseg"][ib], ex["act_colseg"][ib + 1]):
                rr = ex["row_idx"][ex["colseg_ptr"][jj]:ex["colseg_ptr"][jj + 1]]
                assert np.all(rr >= ib * ti) and np.all(rr < min((ib + 1) * ti, a.n_rows))
    with pytest.raises(orc.ConfigError):
        orc.Tiled(orc.make_diag(np.ones(3)), 0, 4)


def test_maspmm_identity_and_zero(orc):  # :221-237
    b = np.asfortranarray(np.random.default_rng(0).uniform(-1, 1, (8, 5)))
    for ti in (1, 3, 8):
        assert np.array_equal(orc.maspmm(orc.Tiled(orc.make_diag(np.ones(8)), ti, 2), b), b)
    zero = orc.Csr.from_triplets(8, 8, [], [], [])
    assert np.all(orc.maspmm(orc.Tiled(zero, 4, 2), b) == 0.0)


def test_maspmm_accumulates(orc):  # :239-248
    a = orc.random_csr(10, 10, 0.4, 17)
    b = np.random.default_rng(1).uniform(-1, 1, (10, 4))
    t = orc.Tiled(a, 3, 2)
    c = orc.maspmm(t, b)
    c = orc.maspmm(t, b, c)
    assert rel_fro(c, 2.0 * orc.naive_spmm(a, b)) <= 1e-14


def test_maspmm_equals_naive_across_tilings(orc):  # :250-263
    a = orc.random_csr(200, 200, 0.05, 42)
    b = orc.fill_gaussian(200, 32, 9, 0)
    want = orc.naive_spmm(a, b)
    for ti, tk in ((1, 1), (7, 8), (64, 64), (200, 32)):
        assert rel_fro(orc.maspmm(orc.Tiled(a, ti, tk), b), want) <= 1e-13


def test_maspmm_linear(orc):  # :265-281
    a = orc.random_symmetric(60, 0.1, 5)
    t = orc.Tiled(a, 16, 4)
    g = np.random.default_rng(2)
    b1, b2 = g.uniform(-1, 1, (60, 8)), g.uniform(-1, 1, (60, 8))
    lhs = orc.maspmm(t, 0.37 * b1 - 2.25 * b2)
    rhs = 0.37 * orc.maspmm(t, b1) - 2.25 * orc.maspmm(t, b2)
    assert rel_fro(lhs, rhs) <= 1e-12


def test_maspmm_bitwise_deterministic(orc):  # :283-295
    a = orc.random_csr(123, 123, 0.08, 77)
    t = orc.Tiled(a, 32, 8)
    b = orc.fill_gaussian(123, 17, 4, 2)
    orc.set_threads(1)
    c1 = orc.maspmm(t, b)
    orc.set_threads(4)
    c2 = orc.maspmm(t, b)
    orc.set_threads(orc.max_threads())
    assert np.array_equal(c1, c2)


def test_maspmm_k0_and_shape_errors(orc):  # :297-309
    t = orc.Tiled(orc.make_diag(np.ones(6)), 2, 4)
    orc.maspmm_shapes(t, (6, 0, 4), (6, 0, 4))
    with pytest.raises(orc.DimensionError):
        orc.maspmm_shapes(t, (5, 3, 4), (6, 3, 4))
    with pytest.raises(orc.DimensionError):
        orc.maspmm_shapes(t, (6, 3, 2), (6, 3, 4))


def test_tiled_maspmm_bitwise_equals_row_order_accumulation(orc):
    # The property the GPU parity rests on: maspmm accumulates each
    # output element in ascending column order, i.e. exactly naive_spmm's CSR order.
    for seed in range(5):
        a = orc.random_csr(150, 150, 0.06, 900 + seed)
        b = orc.fill_gaussian(150, 9, seed, 0)
        for ti, tk in ((1, 1), (7, 8), (64, 64), (256, 64)):
            assert np.array_equal(orc.maspmm(orc.Tiled(a, ti, tk), b), orc.naive_spmm(a, b))


# ----------------------------------------------------- acceptance criteria ---
def test_acceptance4_kernel_equivalence(orc, golden_dir):  # acceptance.cpp:196-245
    mats = []
    rng = orc.MT19937_64(4242)
    for i in range(20):
        n = 50 + rng() % 251
        density = 0.01 + 0.09 * rng.uniform(0.0, 1.0)
        if i % 5 == 4:
            m = 40 + rng() % 100
            mats.append(orc.random_csr(n, m, density, 100 + i))
        else:
            mats.append(orc.random_symmetric(n, density, 100 + i))
    for name in ("laplacian2d_30", "arrow_ints", "banded_mixed"):
        mats.append(load_fixture(orc, golden_dir, name))
    worst, cases = 0.0, 0
    for a in mats:
        for k in (1, 8, 32, 128):
            b = orc.fill_gaussian(a.n_cols, k, 31 + cases, 0)
            want = orc.naive_spmm(a, b)
            for ti, tk in ((1, 1), (7, 8), (64, 64), (256, 64)):
                got = orc.maspmm(orc.Tiled(a, ti, tk), b)
                worst = max(worst, np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))
                cases += 1
    assert cases == 368 and worst <= 1e-13


def test_acceptance5_clenshaw_equivalence(orc):  # acceptance.cpp:249-306
    worst = 0.0
    for n in (60, 130, 200):
        a = orc.random_symmetric(n, 0.08, 600 + n)
        ev = np.linalg.eigvalsh(a.to_dense())
        f = orc.build_filter(ev[n // 4], ev[n // 2], (ev[0] - 0.1, ev[-1] + 0.1), 60, 0.5)
        t = orc.Tiled(a, 32, 8)
        x = orc.fill_gaussian(n, 5, n, 1)
        for degree in (10, 35, 60):
            want = orc.forward_filter_apply(f, a.to_dense(), x, degree)
            worst = max(worst, rel_fro(orc.clenshaw_apply(f, t, x, degree), want))
    assert worst <= 1e-11
    rng = orc.MT19937_64(5)
    diag = [rng.uniform(-0.9, 0.9) for _ in range(150)]
    t = orc.Tiled(orc.make_diag(diag), 64, 16)
    f = orc.build_filter(-0.4, 0.3, (-1.0, 1.0), 50, 0.5)
    x = orc.fill_gaussian(150, 4, 3, 2)
    got = orc.clenshaw_apply(f, t, x, 50)
    want = np.array([orc.eval_filter_scalar(f, d, 50) for d in diag])[:, None] * x
    assert rel_fro(got, want) <= 1e-12


def test_acceptance7_trace_estimate(orc):  # acceptance.cpp:360-392
    good = total = 0
    for count in (5, 50, 200):
        rng = orc.MT19937_64(count)
        d = []
        for i in range(1000):
            if i < count:
                d.append(rng.uniform(0.05, 0.95))
            else:
                v = rng.uniform(2.0, 6.0)
                d.append(v if rng.bernoulli(0.5) else -v)
        t = orc.Tiled(orc.make_diag(d), 256, 64)
        f = orc.build_filter(0.0, 1.0, (-6.5, 6.5), 400, 0.5)
        for seed in range(20):
            c = math.ceil(orc.estimate_eigcount(t, f, 40, seed))
            total += 1
            good += 0.8 * count <= c <= 1.2 * count
    assert good * 10 >= total * 9


def test_golden_fixture_outputs_reproduce(orc, golden_dir):
    z = np.load(f"{golden_dir}/clenshaw_golden.npz")
    for name in ("laplacian2d_30", "arrow_ints", "banded_mixed"):
        if f"{name}/x" not in z:
            continue
        a = load_fixture(orc, golden_dir, name)
        l1, l2, kmax, lo, hi, b0, b1 = z[f"{name}/l1l2"]
        f = orc.build_filter(lo, hi, (b0, b1), int(kmax), 0.5)
        assert np.array_equal(f.coeffs, z[f"{name}/coeffs"])
        t = orc.Tiled(a, 256, 64)
        for d in (0, 1, 2, 3, 17, 40):
            assert np.array_equal(orc.clenshaw_apply(f, t, z[f"{name}/x"], d), z[f"{name}/deg{d}"])


# ------------------------------------------- complex128: real-embedding pin ---
def test_complex_oracle_pinned_by_real_embedding(orc):
    # No reference exists for complex Hermitian input. The complex
    # restatement is pinned by the real embedding S = [[A, -B], [B, A]] of H = A + iB:
    # rho(S) [Re X; Im X] = [Re rho(H) X; Im rho(H) X].
    rng = np.random.default_rng(7)
    n, q = 120, 5
    mask = np.triu(rng.random((n, n)) < 0.06)
    h = np.where(mask, rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), 0)
    h = h + np.conj(np.triu(h, 1)).T
    h[np.diag_indices(n)] = h[np.diag_indices(n)].real
    s = np.block([[h.real, -h.imag], [h.imag, h.real]])

    def csr_of(d):
        r, c = np.nonzero(d)
        return orc.Csr(d.shape[0], d.shape[1],
                       np.concatenate([[0], np.cumsum(np.bincount(r, minlength=d.shape[0]))]).astype(np.int64),
                       c.astype(np.int64), d[r, c])

    hc, sc = csr_of(h), csr_of(s)
    ev = np.linalg.eigvalsh(h)
    bounds = (ev[0] - 0.1, ev[-1] + 0.1)
    f = orc.build_filter(ev[30], ev[60], bounds, 50, 0.5)
    x = rng.standard_normal((n, q)) + 1j * rng.standard_normal((n, q))
    for d in (0, 1, 2, 7, 50):
        got = orc.clenshaw_apply(f, orc.Tiled(hc, 256, 64), x, d)
        emb = orc.clenshaw_apply(f, orc.Tiled(sc, 256, 64), np.vstack([x.real, x.imag]), d)
        assert rel_fro(got, emb[:n] + 1j * emb[n:]) <= 1e-12
    # and the eigenvalues of S are those of H, each doubled
    assert np.allclose(np.linalg.eigvalsh(s)[::2], ev, atol=1e-10)
