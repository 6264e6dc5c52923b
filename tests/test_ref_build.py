"""The oracle restatement against the REFERENCE's own filter-path sources, bit for bit.

oracle/_ref/libadapoly_ref.so is proj/src/cheb_filter.cpp plus the headers it includes (csr_matrix,
tiled_matrix, philox, cheb_filter, types), compiled where they lie under /root/reference against a
minimal Eigen stand-in (oracle/eigen_standin: Eigen is absent from this image; this path only uses
elementwise array arithmetic, which the stand-in evaluates one individually rounded operation at a
time, as Eigen does). So the loops, orders, tilings, index arithmetic and libm calls below are the
reference's own text; what the stand-in supplies is storage and elementwise + - *.

Every function of the path the oracle restates is compared exactly: Philox fills, build_filter (both
dampings), csr_to_tiled + maspmm over tile shapes, clenshaw_apply over degrees / widths / tilings
(including trailing-zero coefficients and degrees 0-2), csr_spmv, naive_spmm, eval_filter_scalar,
initial_degree, adaptive_degree -- on random operators and the reference's own .mtx fixtures.
"""
import os

import numpy as np
import pytest

from oracle import oracle as orc
from oracle import ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (no /root/reference here)")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixture(name):
    z = np.load(os.path.join(GOLDEN, name))
    return orc.Csr(int(z["n_rows"]), int(z["n_cols"]), z["row_ptr"], z["col_idx"], z["values"])


def operators():
    yield "rand200", orc.random_symmetric(200, 0.05, 31)
    yield "rand97", orc.random_symmetric(97, 0.2, 7)
    yield "rand513", orc.random_symmetric(513, 0.01, 5)
    for f in ("fixture_arrow_ints.npz", "fixture_banded_mixed.npz", "fixture_laplacian2d_30.npz"):
        yield f, fixture(f)


def test_philox_fills_bitwise():
    for n, q, seed, stream in ((17, 3, 0, 0), (64, 5, 12345, 2), (1000, 2, 2 ** 40 + 3, 1), (1, 1, 7, 3)):
        assert np.array_equal(orc.fill_gaussian(n, q, seed, stream), ref.fill_gaussian(n, q, seed, stream))
        assert np.array_equal(orc.fill_rademacher(n, q, seed, stream), ref.fill_rademacher(n, q, seed, stream))


@pytest.mark.parametrize("damping", ["lanczos", "jackson"])
def test_build_filter_bitwise(damping):
    for a, b, bounds, k, m in ((0.1, 0.3, (-1.0, 2.0), 40, 0.5), (5.2, 5.85, (0.0, 13.0), 500, 0.5),
                               (-1.0, 1.0, (-1.0, 1.0), 7, 2.0), (0.3, 0.32, (-5.9, 8.6), 1255, 0.5),
                               (-0.5, 0.5, (-2.0, 2.0), 33, 0.0)):
        f = orc.build_filter(a, b, bounds, k, m, damping)
        c, l1, l2, al, be = ref.build_filter(a, b, bounds, k, m, damping)
        assert np.array_equal(f.coeffs, c) and (f.l1, f.l2, f.alpha, f.beta) == (l1, l2, al, be)


def test_maspmm_bitwise_over_tilings():
    rng = np.random.default_rng(0)
    for name, a in operators():
        for t_i, t_k in ((256, 64), (1, 1), (7, 3), (64, 256), (1000, 5)):
            for k in (1, 4, 65):
                b = rng.standard_normal((a.n_cols, k))
                c0 = rng.standard_normal((a.n_rows, k))
                want = ref.maspmm(a, t_i, t_k, b, c0)
                got = orc.maspmm(orc.Tiled(a, t_i, t_k), np.asfortranarray(b), np.asfortranarray(c0.copy()))
                assert np.array_equal(got, want), (name, t_i, t_k, k)


def test_spmv_and_naive_spmm_bitwise():
    rng = np.random.default_rng(1)
    for name, a in operators():
        x = rng.standard_normal(a.n_cols)
        assert np.array_equal(orc.csr_spmv(a, x), ref.csr_spmv(a, x)), name
        b = rng.standard_normal((a.n_cols, 9))
        assert np.array_equal(orc.naive_spmm(a, b), ref.naive_spmm(a, b)), name


def test_clenshaw_apply_bitwise():
    rng = np.random.default_rng(2)
    for name, a in operators():
        if a.n_rows != a.n_cols:
            continue
        spec = np.linalg.eigvalsh(a.to_dense())
        bounds = (spec[0] - 0.1, spec[-1] + 0.1)
        lo, hi = spec[len(spec) // 3], spec[len(spec) // 2]
        f = orc.build_filter(lo, hi, bounds, 60, 0.5)
        for t_i, t_k in ((256, 64), (5, 3), (64, 7)):
            t = orc.Tiled(a, t_i, t_k)
            for q in (1, 3, 64, 70):
                x = rng.standard_normal((a.n_rows, q))
                for degree in (0, 1, 2, 3, 17, 60):
                    cnt = [0]
                    got = orc.clenshaw_apply(f, t, x, degree, cnt)
                    want, wcnt = ref.clenshaw_apply(f.coeffs, f.k_max, f.l1, f.l2, a, t_i, t_k, x, degree)
                    assert np.array_equal(got, want), (name, t_i, t_k, q, degree)
                    assert cnt[0] == wcnt
    # trailing exactly-zero coefficients reduce the degree (cheb_filter.cpp:141-142)
    a = orc.random_symmetric(120, 0.1, 3)
    f = orc.build_filter(-0.25, 0.3, (-8.0, 8.0), 21, 0.5)
    f.coeffs[19:] = 0.0
    x = rng.standard_normal((120, 5))
    cnt = [0]
    got = orc.clenshaw_apply(f, orc.Tiled(a, 256, 64), x, 21, cnt)
    want, wcnt = ref.clenshaw_apply(f.coeffs, f.k_max, f.l1, f.l2, a, 256, 64, x, 21)
    assert np.array_equal(got, want) and cnt[0] == wcnt == 18 * 5


def test_scalar_filter_and_degrees_bitwise():
    rng = np.random.default_rng(3)
    f = orc.build_filter(0.2, 0.5, (-1.0, 3.0), 80, 0.5)
    x = np.concatenate([rng.uniform(-1.5, 3.5, 200), [-1.0, 3.0, 0.2, 0.5]])
    for degree in (0, 1, 2, 41, 80):
        got, gc = orc.eval_filter_scalar(f, x, degree)
        want, wc = ref.eval_filter(f.coeffs, f.k_max, f.l1, f.l2, x, degree)
        assert np.array_equal(got, want) and gc == wc
    for al, be, c in ((1.0, 0.9, 1.4), (0.5, 0.4999, 1.4), (3.0, 0.1, 3.5)):
        assert orc.initial_degree(al, be, c) == ref.initial_degree(al, be, c)
    ritz = np.sort(rng.uniform(-1.0, 3.0, 40))
    for e_i in (1, 5, 20, 40):
        for tau in (1e-1, 1e-3, 1e-8):
            assert orc.adaptive_degree(f, ritz, e_i, tau) == ref.adaptive_degree(f.coeffs, f.k_max, f.l1, f.l2, ritz,
                                                                                 e_i, tau)


def test_config1_full_size_bitwise():
    # BASELINE.json configs[0] (the reference's own CPU-runnable case) at full size: 40^3 7-point Laplacian +
    # potential, block 64, the configuration's initial degree -- oracle restatement vs the reference's sources
    from paper_2604_00914_b200 import configs

    configs.set_rng(orc.uniform_range, orc.gaussian_range)  # the oracle's Philox: no product library needed
    cfg = configs.CONFIGS["c1"]
    a = cfg.operator()
    oa = orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    k = configs.filter_degree(cfg)
    f = orc.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, int(np.ceil(2.5 * k)), 0.5)
    x = orc.fill_gaussian(a.n_rows, cfg.q, 0, 0)
    got = orc.clenshaw_apply(f, orc.Tiled(oa, 256, 64), x, k)
    want, _ = ref.clenshaw_apply(f.coeffs, f.k_max, f.l1, f.l2, oa, 256, 64, x, k)
    assert np.array_equal(got, want)
