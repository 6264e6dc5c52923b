"""GPU parity: the CUDA path through the C-ABI vs the pinned CPU oracle.

The bar is BITWISE equality: the kernel accumulates every
output element in ascending column order with unfused IEEE multiplies and adds
in the reference's expression order, exactly like the reference's maspmm +
Eigen array updates (proj/include/adapoly/tiled_matrix.hpp:205,
proj/src/cheb_filter.cpp:162-177). The north-star tolerance (1e-12 relative
Frobenius per degree) is therefore checked as exact equality.
"""
import numpy as np
import pytest

import paper_2604_00914_b200 as adp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = adp.Context(0)
    yield c
    c.close()


def dev(ctx, a):
    return adp.DeviceCsr(adp.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), ctx)


def same_filter(orc, a, b, bounds, k, m=0.5):
    return adp.build_filter(a, b, bounds, k, m), orc.build_filter(a, b, bounds, k, m)


def assert_bitwise(got, want):
    assert got.shape == want.shape
    if not np.array_equal(got, want):
        diff = np.abs(got - want)
        i = np.unravel_index(np.argmax(diff), diff.shape)
        rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
        raise AssertionError(f"not bitwise equal: max |diff| {diff.max():.3e} at {i}, rel fro {rel:.3e}")


# ------------------------------------------------------------ golden files ---
def test_golden_fixtures(ctx, golden_dir):
    z = np.load(f"{golden_dir}/clenshaw_golden.npz")
    for name in ("laplacian2d_30", "arrow_ints", "banded_mixed"):
        fx = np.load(f"{golden_dir}/fixture_{name}.npz")
        a = adp.DeviceCsr(adp.CsrMatrix(int(fx["n_rows"]), int(fx["n_cols"]), fx["row_ptr"], fx["col_idx"],
                                        fx["values"]), ctx)
        l1, l2, kmax, lo, hi, b0, b1 = z[f"{name}/l1l2"]
        f = adp.build_filter(lo, hi, (b0, b1), int(kmax), 0.5)
        assert np.array_equal(f.coeffs, z[f"{name}/coeffs"])
        for d in (0, 1, 2, 3, 17, 40):
            assert_bitwise(adp.clenshaw_apply(f, a, z[f"{name}/x"], d), z[f"{name}/deg{d}"])


# --------------------------------------------- reference hot-path test cases ---
@pytest.mark.parametrize("q", [1, 2, 3, 5, 6, 8, 16, 17, 30, 33, 64, 65, 128, 130, 256, 266, 290, 362, 384, 520, 1024])
def test_clenshaw_bitwise_widths(ctx, orc, q):
    # random_symmetric(80, 0.1, 31) -- the matrix of test_cheb_filter.cpp:225-240
    a = orc.random_symmetric(80, 0.1, 31)
    spec = np.linalg.eigvalsh(a.to_dense())
    f, g = same_filter(orc, spec[10], spec[50], (spec[0] - 0.1, spec[-1] + 0.1), 60)
    da, t = dev(ctx, a), orc.Tiled(a, 16, 8)
    x = orc.fill_gaussian(80, q, 77, 3)
    for degree in (0, 1, 2, 3, 25, 60):
        s1, s2 = [0], [0]
        assert_bitwise(adp.clenshaw_apply(f, da, x, degree, s1), orc.clenshaw_apply(g, t, x, degree, s2))
        assert s1[0] == s2[0]


def test_clenshaw_diagonal_and_identity(ctx, orc):
    rng = orc.MT19937_64(3)
    diag = [rng.uniform(-0.95, 0.95) for _ in range(40)]
    a = orc.make_diag(diag)
    f, g = same_filter(orc, -0.3, 0.5, (-1.0, 1.0), 35)
    x = orc.fill_gaussian(40, 3, 5, 1)
    for d in (1, 2, 7, 35):
        assert_bitwise(adp.clenshaw_apply(f, dev(ctx, a), x, d), orc.clenshaw_apply(g, orc.Tiled(a, 16, 4), x, d))
    # full-interval filter returns X exactly with no products (test_cheb_filter.cpp:211-223)
    a = orc.random_symmetric(30, 0.2, 9)
    f = adp.build_filter(-40.0, 40.0, (-40.0, 40.0), 20, 0.5)
    x = orc.fill_gaussian(30, 4, 2, 0)
    spmv = [0]
    assert np.array_equal(adp.clenshaw_apply(f, dev(ctx, a), x, 20, spmv), x) and spmv[0] == 0


def test_clenshaw_trailing_zero_and_accounting(ctx, orc):
    a = orc.make_diag([0.1, -0.4, 0.7, 0.2])
    f, g = same_filter(orc, -0.5, 0.5, (-1.0, 1.0), 5, 0.0)
    f.coeffs = g.coeffs = np.array([0.3, 0.5, 0.2, 0.0, 0.0, 0.0])
    x = orc.fill_gaussian(4, 2, 1, 0)
    s = [0]
    assert_bitwise(adp.clenshaw_apply(f, dev(ctx, a), x, 5, s), orc.clenshaw_apply(g, orc.Tiled(a, 2, 2), x, 5))
    assert s[0] == 4
    a = orc.random_symmetric(24, 0.3, 12)
    f = adp.build_filter(-2.0, 5.0, (-30.0, 30.0), 12, 0.5)
    x = orc.fill_gaussian(24, 5, 8, 2)
    s = [0]
    da = dev(ctx, a)
    adp.clenshaw_apply(f, da, x, 12, s)
    adp.clenshaw_apply(f, da, x, 3, s)
    assert s[0] == 75
    with pytest.raises(adp.ConfigError):
        adp.clenshaw_apply(f, da, x, 13)
    with pytest.raises(adp.ConfigError):
        adp.clenshaw_apply(f, da, x, -1)
    with pytest.raises(adp.DimensionError):
        adp.clenshaw_apply(f, da, x[:20], 3)


def test_acceptance5_matrices_bitwise(ctx, orc):
    for n in (60, 130, 200):
        a = orc.random_symmetric(n, 0.08, 600 + n)
        ev = np.linalg.eigvalsh(a.to_dense())
        f, g = same_filter(orc, ev[n // 4], ev[n // 2], (ev[0] - 0.1, ev[-1] + 0.1), 60)
        x = orc.fill_gaussian(n, 5, n, 1)
        for d in (10, 35, 60):
            assert_bitwise(adp.clenshaw_apply(f, dev(ctx, a), x, d), orc.clenshaw_apply(g, orc.Tiled(a, 32, 8), x, d))


# ------------------------------------------------------------------ maspmm ---
def test_spmm_acceptance4_bitwise(ctx, orc, golden_dir):
    mats = []
    rng = orc.MT19937_64(4242)
    for i in range(20):
        n = 50 + rng() % 251
        density = 0.01 + 0.09 * rng.uniform(0.0, 1.0)
        if i % 5 == 4:
            mats.append(orc.random_csr(n, 40 + rng() % 100, density, 100 + i))
        else:
            mats.append(orc.random_symmetric(n, density, 100 + i))
    for name in ("laplacian2d_30", "arrow_ints", "banded_mixed"):
        z = np.load(f"{golden_dir}/fixture_{name}.npz")
        mats.append(orc.Csr(int(z["n_rows"]), int(z["n_cols"]), z["row_ptr"], z["col_idx"], z["values"]))
    cases = 0
    for a in mats:
        da = dev(ctx, a)
        for k in (1, 8, 32, 128):
            b = orc.fill_gaussian(a.n_cols, k, 31 + cases, 0)
            want = orc.maspmm(orc.Tiled(a, 256, 64), b)
            assert_bitwise(adp.maspmm(da, b), want)
            c0 = orc.fill_gaussian(a.n_rows, k, 5, 5)
            assert_bitwise(adp.maspmm(da, b, c0), orc.maspmm(orc.Tiled(a, 7, 8), b, c0))
            cases += 1
    assert cases == 92


def test_spmm_errors(ctx, orc):
    a = dev(ctx, orc.make_diag(np.ones(6)))
    with pytest.raises(adp.DimensionError):
        adp.maspmm(a, np.zeros((5, 3)))
    assert adp.maspmm(a, np.zeros((6, 0))).shape == (6, 0)


# ------------------------------------------------------------- device API ---
def test_device_api_layouts(ctx, orc):
    a = orc.random_symmetric(300, 0.03, 7)
    spec = np.linalg.eigvalsh(a.to_dense())
    f, g = same_filter(orc, spec[100], spec[140], (spec[0] - 0.1, spec[-1] + 0.1), 30)
    da, t = dev(ctx, a), orc.Tiled(a, 256, 64)
    for q, ldx, ldy, off in [(64, 64, 64, 0), (5, 5, 7, 0), (6, 10, 6, 1), (33, 40, 34, 0), (128, 130, 128, 0)]:
        x = orc.fill_gaussian(300, q, q, 0)
        xt = torch.zeros(300 * ldx + 2, dtype=torch.float64, device="cuda")
        xv = xt[off:off + 300 * ldx].view(300, ldx)[:, :q]
        xv.copy_(torch.from_numpy(np.ascontiguousarray(x)))
        yt = torch.full((300 * ldy + 2,), float("nan"), dtype=torch.float64, device="cuda")
        yv = yt[off:off + 300 * ldy].view(300, ldy)[:, :q]
        for d in (0, 1, 2, 9, 30):
            adp.clenshaw_apply_device(f, da, xv, d, out=yv)
            torch.cuda.synchronize()
            assert_bitwise(yv.cpu().numpy(), orc.clenshaw_apply(g, t, x, d))
        if ldy > q:  # padding columns of the caller's buffer are untouched
            assert torch.isnan(yt[off:off + 300 * ldy].view(300, ldy)[:, q:]).all()


def test_host_row_major_layout(ctx, orc):
    a = orc.random_symmetric(120, 0.05, 3)
    f, g = same_filter(orc, -0.5, 0.2, (-8.0, 8.0), 20)
    x = orc.fill_gaussian(120, 7, 1, 0)
    want = orc.clenshaw_apply(g, orc.Tiled(a, 256, 64), x, 20)
    assert_bitwise(adp.clenshaw_apply(f, dev(ctx, a), np.ascontiguousarray(x), 20, layout="row"), want)


def test_bitwise_deterministic_repeat(ctx, orc):
    a = orc.random_csr(500, 500, 0.02, 77)
    da = dev(ctx, a)
    f = adp.build_filter(-0.5, 0.5, (-10.0, 10.0), 50, 0.5)
    x = orc.fill_gaussian(500, 17, 4, 2)
    r1 = adp.clenshaw_apply(f, da, x, 50)
    r2 = adp.clenshaw_apply(f, da, x, 50)
    assert np.array_equal(r1, r2)


def test_launch_count_is_degree(ctx, orc):
    a = orc.random_symmetric(100, 0.05, 1)
    f = adp.build_filter(-0.5, 0.5, (-10.0, 10.0), 40, 0.5)
    x = torch.zeros(100, 64, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    n0 = ctx.launch_count
    adp.clenshaw_apply_device(f, dev(ctx, a), x, 40, out=y)
    assert ctx.launch_count - n0 == 40  # one fused kernel per degree step


# --------------------------------------------------------------- complex ---
def random_hermitian(n, density, seed):
    rng = np.random.default_rng(seed)
    m = rng.random((n, n)) < density
    m = np.triu(m)
    vals = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = np.where(m, vals, 0)
    h = h + np.conj(np.triu(h, 1)).T
    h[np.diag_indices(n)] = h[np.diag_indices(n)].real
    r, c = np.nonzero(h)
    return adp.CsrMatrix.from_triplets(n, n, r, c, h[r, c])


def test_complex_bitwise_vs_oracle(ctx, orc):
    for n, q in [(90, 3), (150, 16), (200, 40), (256, 130), (210, 150), (180, 200)]:
        h = random_hermitian(n, 0.05, n)
        oh = orc.Csr(h.n_rows, h.n_cols, h.row_ptr, h.col_idx, h.values)
        ev = np.linalg.eigvalsh(h.to_dense())
        f, g = same_filter(orc, ev[n // 3], ev[n // 2], (ev[0] - 0.1, ev[-1] + 0.1), 40)
        rng = np.random.default_rng(q)
        x = np.asfortranarray(rng.standard_normal((n, q)) + 1j * rng.standard_normal((n, q)))
        da, t = adp.DeviceCsr(h, ctx), orc.Tiled(oh, 256, 64)
        for d in (0, 1, 2, 5, 40):
            assert_bitwise(adp.clenshaw_apply(f, da, x, d), orc.clenshaw_apply(g, t, x, d))


def test_int64_row_offsets_path(ctx, orc, monkeypatch):
    # config 5 (nnz > 2^31) needs int64 row offsets; force them on small operators, real and complex
    monkeypatch.setenv("ADP_FORCE_RP64", "1")
    a = orc.random_symmetric(300, 0.03, 17)
    f, g = same_filter(orc, -0.5, 0.5, (-8.0, 8.0), 30)
    t = orc.Tiled(a, 256, 64)
    da = dev(ctx, a)
    for q in (3, 64, 130):
        x = orc.fill_gaussian(300, q, q, 1)
        for d in (1, 2, 30):
            assert_bitwise(adp.clenshaw_apply(f, da, x, d), orc.clenshaw_apply(g, t, x, d))
        assert_bitwise(adp.maspmm(da, x), orc.maspmm(t, x))
    h = random_hermitian(120, 0.05, 3)
    oh = orc.Csr(h.n_rows, h.n_cols, h.row_ptr, h.col_idx, h.values)
    xz = np.asfortranarray(np.random.default_rng(1).standard_normal((120, 33)) + 0j)
    assert_bitwise(adp.clenshaw_apply(f, adp.DeviceCsr(h, ctx), xz, 30),
                   orc.clenshaw_apply(g, orc.Tiled(oh, 256, 64), xz, 30))


# ------------------------------------------------------- full-size configs ---
def test_config1_full_size_bitwise(ctx, orc):
    from paper_2604_00914_b200 import configs

    cfg = configs.CONFIGS["c1"]
    a = cfg.operator()
    k = configs.filter_degree(cfg)
    f, g = same_filter(orc, cfg.window[0], cfg.window[1], cfg.bounds, int(np.ceil(2.5 * k)))
    x = orc.fill_gaussian(a.n_rows, cfg.q, 0, 0)
    oa = orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    got = adp.clenshaw_apply(f, adp.DeviceCsr(a, ctx), x, k)
    assert_bitwise(got, orc.clenshaw_apply(g, orc.Tiled(oa, 256, 64), x, k))
    # BASELINE.json configs[0] at its full size and block width against the REFERENCE's own clenshaw_apply
    # (oracle/_ref: its sources compiled against the Eigen stand-in), on the reference's own Philox block
    from oracle import ref

    if ref.available():
        coeffs, l1, l2, _, _ = ref.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, int(np.ceil(2.5 * k)), 0.5)
        assert np.array_equal(coeffs, f.coeff_array())
        xr = ref.fill_gaussian(a.n_rows, cfg.q, 0, 0)
        assert np.array_equal(xr, x)
        want, _ = ref.clenshaw_apply(coeffs, len(coeffs) - 1, l1, l2, oa, 256, 64, xr, k)
        assert_bitwise(got, want)


@pytest.mark.slow
def test_config2_full_size_bitwise_low_degree(ctx, orc):
    # n = 1e6, q = 256 (2 GB per block): a few degree steps vs the oracle, bitwise, plus repeatability.
    from paper_2604_00914_b200 import configs

    cfg = configs.CONFIGS["c2"]
    a = cfg.operator()
    f, g = same_filter(orc, cfg.window[0], cfg.window[1], cfg.bounds, 40)
    x = orc.fill_gaussian(a.n_rows, cfg.q, 0, 0)
    oa = orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    da = adp.DeviceCsr(a, ctx)
    got = adp.clenshaw_apply(f, da, x, 4)
    assert_bitwise(got, orc.clenshaw_apply(g, orc.Tiled(oa, 256, 64), x, 4))
    assert np.array_equal(adp.clenshaw_apply(f, da, x, 4), got)


# ------------------------------------------------- every kernel variant ---
# Every kernel family (adp_ctx_set_tuning: 1 row, 2 lean, 3 line, 4 cube,
# 5 plane sweep, 6 / 7 band blocks) must be bitwise equal to the oracle: they only reorganise
# loads, never the per-element arithmetic. Stencil operators exercise the
# shifted-pattern blocks (and their irregular faces) and the plane sweep
# (grids not multiples of its 8 x 8 tiles), a random matrix the row-by-row
# fallbacks.
VARIANTS = [0, 1, 2, 3, 4, 5, 6, 7]


@pytest.mark.parametrize("kind", ["lap7", "lap27", "random", "hermitian", "band"])
def test_kernel_variants_bitwise(ctx, orc, kind):
    from paper_2604_00914_b200 import configs

    if kind == "band":  # config 5's structure (band + random off-band entries): the line kernel's band blocks
        a = configs.random_banded_hermitian(600, 40, 4, seed=2)
    elif kind == "lap7":
        a = configs.laplacian7_potential(11, -2.0, 2.0, seed=3)
    elif kind == "lap27":
        a = configs.dft_like_27pt(9, n_centres=4, seed=1)
    elif kind == "random":
        a = adp.CsrMatrix(*(lambda m: (m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values))(orc.random_symmetric(700, 0.01, 5)))
    else:
        a = random_hermitian(300, 0.03, 9)
    n = a.n_rows
    oa = orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    t = orc.Tiled(oa, 256, 64)
    dense_bounds = (-30.0, 30.0)
    f, g = same_filter(orc, -0.3, 0.4, dense_bounds, 12)
    da = adp.DeviceCsr(a, ctx)
    rng = np.random.default_rng(n)
    for q in (64, 256):
        x = rng.standard_normal((n, q))
        if a.is_complex:
            x = x + 1j * rng.standard_normal((n, q))
        x = np.asfortranarray(x)
        want = {d: orc.clenshaw_apply(g, t, x, d) for d in (1, 2, 5, 12)}
        want_spmm = None if a.is_complex else orc.maspmm(t, x)  # the oracle's maspmm is real-only
        try:
            for v in VARIANTS:
                ctx.set_tuning(v)
                for d, w in want.items():
                    try:
                        assert_bitwise(adp.clenshaw_apply(f, da, x, d), w)
                    except AssertionError as e:
                        raise AssertionError(f"variant {v} degree {d} q {q}: {e}") from None
                if want_spmm is not None:
                    assert_bitwise(adp.maspmm(da, x), want_spmm)
        finally:
            ctx.set_tuning(0)


def test_auto_line_kernel_ragged_widths(ctx, orc):
    # the automatic line kernel (27-point stencil: long rows) on ragged and odd widths: full 64-vector
    # panels + one masked launch, odd q through the padded leading dimension -- bitwise vs the oracle
    from paper_2604_00914_b200 import configs

    a = configs.dft_like_27pt(9, n_centres=4, seed=2)
    n = a.n_rows
    oa = orc.Csr(n, n, a.row_ptr, a.col_idx, a.values)
    t = orc.Tiled(oa, 256, 64)
    f, g = same_filter(orc, -0.3, 0.4, (-30.0, 30.0), 9)
    da = adp.DeviceCsr(a, ctx)
    rng = np.random.default_rng(5)
    for q in (20, 33, 101, 150, 129):
        x = np.asfortranarray(rng.standard_normal((n, q)))
        for d in (1, 2, 9):
            assert_bitwise(adp.clenshaw_apply(f, da, x, d), orc.clenshaw_apply(g, t, x, d))
        assert_bitwise(adp.maspmm(da, x), orc.maspmm(t, x))


# --------------------------------------------- operators created from device arrays ---
def _torch_csr(a):
    return (torch.from_numpy(np.asarray(a.row_ptr, np.int64)).cuda(),
            torch.from_numpy(np.asarray(a.col_idx, np.int32)).cuda(),
            torch.from_numpy(np.asarray(a.values)).cuda())


def test_device_created_operator_bitwise(ctx, orc, monkeypatch):
    # adp_csr_create_device: same results as the host-created operator, int32 and forced int64 offsets,
    # real and complex, including the line kernel (27-point stencil: its plan needs the lazy host copy)
    from paper_2604_00914_b200 import configs

    lap27 = configs.dft_like_27pt(9, n_centres=4, seed=1)
    herm = random_hermitian(150, 0.05, 4)
    for force in ("0", "1"):
        monkeypatch.setenv("ADP_FORCE_RP64", force)
        for a in (lap27, herm):
            n = a.n_rows
            oa = orc.Csr(n, n, a.row_ptr, a.col_idx, a.values)
            f, g = same_filter(orc, -0.3, 0.4, (-30.0, 30.0), 12)
            da = adp.DeviceCsr.from_device(n, n, *_torch_csr(a), ctx=ctx)
            assert da.nnz == a.nnz and da.is_complex == a.is_complex
            rng = np.random.default_rng(n)
            for q in (17, 128):
                x = rng.standard_normal((n, q))
                if a.is_complex:
                    x = x + 1j * rng.standard_normal((n, q))
                x = np.asfortranarray(x)
                for d in (1, 2, 12):
                    assert_bitwise(adp.clenshaw_apply(f, da, x, d), orc.clenshaw_apply(g, orc.Tiled(oa, 256, 64), x, d))
            da.close()


def test_device_created_operator_validation(ctx):
    # CsrMatrix::validate (csr_matrix.hpp:101-116) on the device: DimensionError for each broken invariant
    a = adp.CsrMatrix.from_triplets(4, 4, [0, 0, 1, 2, 3], [0, 2, 1, 2, 3], [1.0, 2.0, 3.0, 4.0, 5.0])
    rp, ci, v = _torch_csr(a)
    ok = adp.DeviceCsr.from_device(4, 4, rp, ci, v, ctx=ctx)
    ok.close()
    bad_cols = [ci.clone(), ci.clone(), ci.clone()]
    bad_cols[0][1] = 0  # not strictly increasing
    bad_cols[1][4] = 4  # out of range
    bad_cols[2][0] = -1
    for c in bad_cols:
        with pytest.raises(adp.DimensionError):
            adp.DeviceCsr.from_device(4, 4, rp, c, v, ctx=ctx)
    bad_rp = rp.clone()
    bad_rp[2] = 1  # decreasing
    with pytest.raises(adp.DimensionError):
        adp.DeviceCsr.from_device(4, 4, bad_rp, ci, v, ctx=ctx)
    with pytest.raises(adp.ConfigError):
        adp.DeviceCsr.from_device(4, 4, rp, ci.to(torch.int64), v, ctx=ctx)
    with pytest.raises(adp.DimensionError):
        adp.DeviceCsr.from_device(5, 5, rp, ci, v, ctx=ctx)


def test_gpu_bitwise_vs_reference_sources(ctx, orc, golden_dir):
    # The GPU path against the REFERENCE's own clenshaw_apply / maspmm source text (oracle/_ref: compiled
    # from /root/reference against the Eigen stand-in, prebuilt on this box), not only against the oracle
    # restatement: random operators, the reference's .mtx fixtures, a 7-point stencil (plane-sweep kernel).
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    from paper_2604_00914_b200 import configs

    rng = np.random.default_rng(11)
    ops = [orc.random_symmetric(300, 0.04, 5), orc.random_symmetric(1025, 0.004, 6)]
    for name in ("arrow_ints", "banded_mixed", "laplacian2d_30"):
        z = np.load(f"{golden_dir}/fixture_{name}.npz")
        if int(z["n_rows"]) == int(z["n_cols"]):
            ops.append(orc.Csr(int(z["n_rows"]), int(z["n_cols"]), z["row_ptr"], z["col_idx"], z["values"]))
    s = configs.laplacian7_potential(12, -2.0, 2.0, seed=3)
    ops.append(orc.Csr(s.n_rows, s.n_cols, s.row_ptr, s.col_idx, s.values))
    for a in ops:
        bound = float(np.abs(a.to_dense()).sum(axis=1).max()) + 0.5
        f = adp.build_filter(-0.3 * bound, 0.1 * bound, (-bound, bound), 48, 0.5)
        coeffs, l1, l2, _, _ = ref.build_filter(-0.3 * bound, 0.1 * bound, (-bound, bound), 48, 0.5)
        assert np.array_equal(f.coeff_array(), coeffs) and (f.l1, f.l2) == (l1, l2)
        da = dev(ctx, a)
        for q in (1, 7, 64, 96):
            x = rng.standard_normal((a.n_rows, q))
            for degree in (1, 2, 9, 48):
                got = adp.clenshaw_apply(f, da, x, degree)
                want, _ = ref.clenshaw_apply(coeffs, 48, l1, l2, a, 256, 64, x, degree)
                assert_bitwise(got, want)
            b = rng.standard_normal((a.n_cols, q))
            assert_bitwise(adp.maspmm(da, b), ref.maspmm(a, 256, 64, b))
        da.close()
