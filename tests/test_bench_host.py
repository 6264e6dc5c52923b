"""Host-side pieces of bench.py and the configuration generators (CPU only)."""
import numpy as np

from paper_2604_00914_b200 import configs


def test_oracle_rng_builds_the_same_operators(orc):
    # bench.py's reference arm builds its operator with the oracle's Philox (configs.set_rng) so that it
    # never maps the product library: the operators must be bitwise the product generator's
    orc.build()
    builders = [lambda: configs.laplacian7_potential(8, -2.0, 2.0, seed=3), lambda: configs.dft_like_27pt(8, 4, 1),
                lambda: configs.peierls_lattice(6), lambda: configs.random_banded_hermitian(60, 5, 2, seed=1)]
    for build in builders:
        configs.set_rng()
        a = build()
        configs.set_rng(orc.uniform_range, orc.gaussian_range)
        try:
            b = build()
        finally:
            configs.set_rng()
        assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
        assert np.array_equal(a.values, b.values)


def test_both_arms_print_the_same_config():
    import bench

    cfg = configs.CONFIGS["c4"]
    n, nnz, q, deg = 128 ** 3, 55_742_968, 1024, configs.filter_degree(cfg)
    w = bench.workload("c4", cfg, n, nnz, q, deg, 8, 1)
    assert w == bench.workload("c4", cfg, n, nnz, q, deg, 8, 1)
    assert w["workload"].startswith("c4:") and w["degree"] == 502
    assert w["bytes_per_degree_step"] == nnz * 12 + (n + 1) * 4 + 4 * n * q * 8  # 69.40 GB
    assert abs(w["bytes_per_degree_step"] - 69.40e9) < 0.01e9


def test_plane_ranges():
    import bench

    for planes, world in ((128, 8), (100, 3), (7, 2)):
        r = bench.plane_ranges(planes * 50, 50, world)
        assert r[0][0] == 0 and r[-1][1] == planes * 50
        assert all(b == c for (_, b), (c, _) in zip(r, r[1:]))
        assert all(lo % 50 == 0 and hi % 50 == 0 and hi > lo for lo, hi in r)


def test_c1t_window_is_small():
    cfg = configs.CONFIGS["c1t"]
    a = cfg.operator()
    assert a.n_rows == 16 ** 3
    assert cfg.window[1] - cfg.window[0] < 0.05
