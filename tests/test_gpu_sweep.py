"""The plane-sweep stencil kernel (csrc/cheb_sweep.cu) against the oracle, bitwise.

The kernel re-encodes a constant-coefficient 7- or 27-point operator (one value
per offset, the diagonal per row) after verifying that encoding entry by entry
against the CSR, and streams halo tiles of W plane by plane through shared
memory. Its products still accumulate per output in ascending column order with
unfused multiplies and adds (proj/include/adapoly/tiled_matrix.hpp:200-205,
proj/src/cheb_filter.cpp:167-177), so the bar is bitwise equality with the
oracle -- on grids that are not multiples of its 8 x 8 tiles, ragged and odd
block widths, padded leading dimensions and more (panel, tile) items than SMs.
"""
import numpy as np
import pytest

import paper_2604_00914_b200 as adp
from paper_2604_00914_b200 import configs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SWEEP = 5  # adp_ctx_last_step_kernel family code


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = adp.Context(0)
    yield c
    c.close()


def grid_operator(kind, nx, ny, nz, seed=0, general=False):
    """A kind-point stencil with a Philox potential. The configs' weights (Mehrstellen 27-point: one value
    per distance class -> the kernel's shared class products; 7-point: all -1 -> subtractions), or with
    ``general`` one distinct value per offset (the kernel's per-offset product path)."""
    offs, ws = configs._twenty_seven_point() if kind == 27 else configs._seven_point()
    if general:
        ws = [-(0.3 + 0.05 * j) for j in range(len(offs))]
    u = adp.philox_uniform(seed, configs.STREAM_POTENTIAL, 0, nx * ny * nz)
    centre = ws[13] if kind == 27 else 6.0
    return configs.stencil_3d(nx, offs, ws, centre - 2.0 + 4.0 * u, ny=ny, nz=nz)


def oracle_apply(orc, a, g, x, d):
    t = orc.Tiled(orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), 256, 64)
    return orc.clenshaw_apply(g, t, np.asfortranarray(x), d)


def assert_bitwise(got, want):
    assert got.shape == want.shape
    if not np.array_equal(got, want):
        diff = np.abs(got - want)
        raise AssertionError(f"not bitwise equal: max |diff| {diff.max():.3e} at "
                             f"{np.unravel_index(np.argmax(diff), diff.shape)}")


def test_stencil_detection(ctx, orc):
    assert adp.DeviceCsr(grid_operator(27, 9, 5, 7), ctx).stencil() == (27, (9, 5, 7))
    assert adp.DeviceCsr(grid_operator(7, 13, 17, 6), ctx).stencil() == (7, (13, 17, 6))
    assert adp.DeviceCsr(configs.laplacian7_potential(40, 0.0, 1.0), ctx).stencil() == (7, (40, 40, 40))
    # not stencils: an off-diagonal value that differs in one row; a missing entry; random sparsity; complex
    a = grid_operator(27, 9, 5, 7)
    v = a.values.copy()
    v[a.row_ptr[100] + 2] *= 1.0000001
    assert adp.DeviceCsr(adp.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, v), ctx).stencil()[0] == 0
    keep = np.ones(a.nnz, bool)
    keep[a.row_ptr[200] + 1] = False
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr))[keep]
    b = adp.CsrMatrix.from_triplets(a.n_rows, a.n_cols, rows, a.col_idx[keep], a.values[keep])
    assert adp.DeviceCsr(b, ctx).stencil()[0] == 0
    r = orc.random_symmetric(500, 0.02, 3)
    assert adp.DeviceCsr(adp.CsrMatrix(r.n_rows, r.n_cols, r.row_ptr, r.col_idx, r.values), ctx).stencil()[0] == 0
    assert adp.DeviceCsr(configs.peierls_lattice(20), ctx).stencil()[0] == 0


@pytest.mark.parametrize("kind,dims,general", [(27, (9, 5, 7), False), (27, (16, 8, 4), False), (27, (10, 11, 3), False),
                                               (7, (13, 17, 6), False), (7, (8, 8, 8), False), (7, (21, 3, 5), False),
                                               (27, (9, 5, 7), True), (7, (13, 17, 6), True)])
def test_sweep_bitwise_shapes(ctx, orc, kind, dims, general):
    a = grid_operator(kind, *dims, seed=sum(dims), general=general)
    da = adp.DeviceCsr(a, ctx)
    assert da.stencil() == (kind, dims)
    bounds = (-12.0, 16.0) if kind == 27 else (-3.0, 15.0)
    f = adp.build_filter(0.2, 0.9, bounds, 24, 0.5)
    g = orc.build_filter(0.2, 0.9, bounds, 24, 0.5)
    rng = np.random.default_rng(a.n_rows)
    for q in (1, 3, 32, 33, 64, 100):
        x = rng.standard_normal((a.n_rows, q))
        for d in (2, 5, 24):
            got = adp.clenshaw_apply(f, da, x, d)
            assert ctx.last_step_kernel == SWEEP
            try:
                assert_bitwise(got, oracle_apply(orc, a, g, x, d))
            except AssertionError as e:
                raise AssertionError(f"q {q} degree {d}: {e}") from None


def test_sweep_many_items_and_fallback_equal(ctx, orc):
    # config 1's 40^3 operator at q = 320: 10 panels x 25 tiles = 250 items > 148 SMs; the lean kernel
    # (family 2) on the same call gives the same bits
    a = configs.laplacian7_potential(40, 0.0, 1.0)
    da = adp.DeviceCsr(a, ctx)
    f = adp.build_filter(5.2, 5.85, (0.0, 13.0), 40, 0.5)
    g = orc.build_filter(5.2, 5.85, (0.0, 13.0), 40, 0.5)
    x = np.random.default_rng(7).standard_normal((a.n_rows, 320))
    got = adp.clenshaw_apply(f, da, x, 9)
    assert ctx.last_step_kernel == SWEEP
    assert_bitwise(got, oracle_apply(orc, a, g, x, 9))
    try:
        ctx.set_tuning(2)
        lean = adp.clenshaw_apply(f, da, x, 9)
        assert ctx.last_step_kernel == 2
    finally:
        ctx.set_tuning(0)
    assert_bitwise(lean, got)


def test_sweep_device_padded_leading_dimensions(ctx, orc):
    a = grid_operator(27, 12, 9, 6, seed=4)
    da = adp.DeviceCsr(a, ctx)
    f = adp.build_filter(0.1, 0.7, (-12.0, 16.0), 16, 0.5)
    g = orc.build_filter(0.1, 0.7, (-12.0, 16.0), 16, 0.5)
    n, q = a.n_rows, 37
    xh = np.random.default_rng(11).standard_normal((n, q))
    xs = torch.zeros(n, 50, dtype=torch.float64, device="cuda")
    xs[:, :q] = torch.from_numpy(xh).cuda()
    outs = torch.full((n, 44), 7.0, dtype=torch.float64, device="cuda")
    adp.clenshaw_apply_device(f, da, xs[:, :q], 16, out=outs[:, :q])
    torch.cuda.synchronize()
    assert ctx.last_step_kernel == SWEEP
    assert_bitwise(outs[:, :q].cpu().numpy(), oracle_apply(orc, a, g, xh, 16))
    assert torch.all(outs[:, q:] == 7.0)  # nothing written past the block's columns
