"""The band-block kernel (csrc/cheb_band.cu) against the oracle, bitwise (config 5's structure).

A warp sweeps the union of R consecutive rows' bands column by column and applies each W row panel to
every row whose band holds it; per row the products still accumulate in CSR order (lower off-band,
band, upper off-band), so the result is bitwise the CSR kernels' / the oracle's -- on complex and real
banded operators, rows at the matrix edges (truncated bands), ragged widths and more row blocks than
one sweep; a matrix with a hole in one row's band falls back to the lean kernel.
"""
import numpy as np
import pytest

import paper_2604_00914_b200 as adp
from paper_2604_00914_b200 import configs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
BAND = 6


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = adp.Context(0)
    yield c
    c.close()


def real_banded(n, hb, off, seed):
    h = configs.random_banded_hermitian(n, hb, off, seed=seed)
    v = h.values.real.copy()
    return adp.CsrMatrix(h.n_rows, h.n_cols, h.row_ptr, h.col_idx, v)


def oracle_apply(orc, a, g, x, d):
    t = orc.Tiled(orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), 256, 64)
    return orc.clenshaw_apply(g, t, np.asfortranarray(x), d)


@pytest.mark.parametrize("kind,n,hb,off", [("c128", 3000, 40, 4), ("c128", 1500, 100, 2), ("f64", 2500, 33, 3)])
@pytest.mark.parametrize("variant", [0, 7])
def test_band_kernel_bitwise(ctx, orc, kind, n, hb, off, variant):
    a = configs.random_banded_hermitian(n, hb, off, seed=n) if kind == "c128" else real_banded(n, hb, off, n)
    da = adp.DeviceCsr(a, ctx)
    f = adp.build_filter(-1.0, 1.5, (-60.0, 60.0), 12, 0.5)
    g = orc.build_filter(-1.0, 1.5, (-60.0, 60.0), 12, 0.5)
    rng = np.random.default_rng(n + hb)
    ctx.set_tuning(variant)
    try:
        for q in (1, 3, 64, 65, 200):
            x = rng.standard_normal((n, q))
            if a.is_complex:
                x = x + 1j * rng.standard_normal((n, q))
            for d in (2, 6, 12):
                got = adp.clenshaw_apply(f, da, x, d)
                assert ctx.last_step_kernel == BAND
                want = oracle_apply(orc, a, g, x, d)
                assert np.array_equal(got, want), (kind, q, d)
    finally:
        ctx.set_tuning(0)


def test_band_hole_falls_back(ctx, orc):
    a = configs.random_banded_hermitian(2000, 40, 2, seed=1)
    # drop one band entry of row 700 (and its mirror, keeping the matrix Hermitian): no longer a full band
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr))
    kill = ((rows == 700) & (a.col_idx == 705)) | ((rows == 705) & (a.col_idx == 700))
    b = adp.CsrMatrix.from_triplets(a.n_rows, a.n_cols, rows[~kill], a.col_idx[~kill], a.values[~kill])
    db = adp.DeviceCsr(b, ctx)
    f = adp.build_filter(-1.0, 1.5, (-60.0, 60.0), 8, 0.5)
    g = orc.build_filter(-1.0, 1.5, (-60.0, 60.0), 8, 0.5)
    x = np.random.default_rng(2).standard_normal((a.n_rows, 64)) + 0j
    got = adp.clenshaw_apply(f, db, x, 8)
    assert ctx.last_step_kernel != BAND
    assert np.array_equal(got, oracle_apply(orc, b, g, x, 8))
