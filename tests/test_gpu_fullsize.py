"""Full-size parity on BASELINE.json's configurations 2, 3 and 4 and config 5's structure (c5s) (GPU).

The oracle cannot run a full n x q block at these sizes in seconds, but the
step kernel computes every column independently: so the GPU result of the
FULL-width block at full n is checked, column pair by column pair, bitwise
against the CPU oracle run on just those two columns at full n. Plus the
size-independent properties: bitwise repeatability, and host-API (column-major,
pinned) == device-API results.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2604_00914_b200 as adp
from paper_2604_00914_b200 import _native, configs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = adp.Context(0)
    yield c
    c.close()


def device_block(ctx, n, q, complex_=False, seed=3):
    """Rademacher entries generated on the device (exact: identical to the host Philox fill)."""
    dt = torch.complex128 if complex_ else torch.float64
    x = torch.empty(n, q, dtype=dt, device="cuda")
    if complex_:
        re = torch.empty(n, q, dtype=torch.float64, device="cuda")
        im = torch.empty(n, q, dtype=torch.float64, device="cuda")
        for t, s in ((re, seed), (im, seed + 1)):
            _native.check(_native.lib().adp_fill_rademacher_device(ctx.h, C.c_void_p(t.data_ptr()), n, q, q, s, 2))
        x = torch.complex(re, im)
    else:
        _native.check(_native.lib().adp_fill_rademacher_device(ctx.h, C.c_void_p(x.data_ptr()), n, q, q, seed, 2))
    torch.cuda.synchronize()
    return x


@pytest.mark.parametrize("name,degree,cols", [("c2", 8, [(0, 2), (130, 132), (254, 256)]),
                                              ("c3", 6, [(0, 2), (383, 384)]),
                                              ("c4", 4, [(0, 2), (1022, 1024)]),
                                              ("c5s", 3, [(0, 1), (200, 201), (383, 384)])])
def test_full_size_columns_bitwise_vs_oracle(ctx, orc, name, degree, cols):
    cfg = configs.CONFIGS[name]
    a = cfg.operator()
    n, q = a.n_rows, cfg.q
    da = adp.DeviceCsr(a, ctx)
    k_max = max(degree, 40)
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, k_max, 0.5)
    g = orc.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, k_max, 0.5)
    x = device_block(ctx, n, q, a.is_complex)
    y = adp.clenshaw_apply_device(f, da, x, degree)
    y2 = adp.clenshaw_apply_device(f, da, x, degree)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)  # bitwise repeatable
    oa = orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    t = orc.Tiled(oa, 256, 64)
    for c0, c1 in cols:
        xs = np.asfortranarray(x[:, c0:c1].cpu().numpy())
        want = orc.clenshaw_apply(g, t, xs, degree)
        got = y[:, c0:c1].cpu().numpy()
        assert np.array_equal(got, want), (name, c0, c1)
    del y, y2, x
    torch.cuda.empty_cache()


def test_host_api_equals_device_api_config2(ctx):
    cfg = configs.CONFIGS["c2"]
    a = cfg.operator()
    da = adp.DeviceCsr(a, ctx)
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, 40, 0.5)
    x = device_block(ctx, a.n_rows, 64)
    yd = adp.clenshaw_apply_device(f, da, x, 5).cpu().numpy()
    yh = adp.clenshaw_apply(f, da, np.asfortranarray(x.cpu().numpy()), 5)
    assert np.array_equal(yd, yh)


# ---- at the bench's own degrees: the driver-run suite checks the exact calls bench.py times ----
# bench.py times clenshaw_apply at each configuration's initial degree k1 (config 2: 7282, config 4:
# 502). The kernel computes columns independently, so the full-width GPU call is checked on column
# pairs against the oracle run on those columns at full n and the same degree -- bitwise (per-step
# bitwise equality makes this expected; here it is measured at the bench's degree).
@pytest.mark.parametrize("name,cols", [("c2", [(0, 2), (254, 256)]), ("c4", [(0, 2), (1022, 1024)])])
def test_bench_degree_columns_bitwise_vs_oracle(ctx, orc, name, cols):
    cfg = configs.CONFIGS[name]
    a = cfg.operator()
    n, q = a.n_rows, cfg.q
    k1 = configs.filter_degree(cfg)
    k_max = int(np.ceil(2.5 * k1))
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, k_max, 0.5)
    g = orc.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, k_max, 0.5)
    da = adp.DeviceCsr(a, ctx)
    x = device_block(ctx, n, q, seed=11)
    y = adp.clenshaw_apply_device(f, da, x, k1)
    torch.cuda.synchronize()
    assert ctx.last_step_kernel == 5  # the plane-sweep kernel, as in the bench
    assert torch.isfinite(y).all()
    orc.set_threads(orc.max_threads())
    t = orc.Tiled(orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), 256, 64)
    for c0, c1 in cols:
        want = orc.clenshaw_apply(g, t, np.asfortranarray(x[:, c0:c1].cpu().numpy()), k1)
        got = y[:, c0:c1].cpu().numpy()
        assert np.array_equal(got, want), (name, k1, c0, c1)
    del x, y
    da.close()
    torch.cuda.empty_cache()


def test_host_api_pipelined_chunks_equal_device_api(ctx):
    # blocks >= 1 GB go through the host API in column chunks whose copies overlap the previous chunk's
    # filter (capi.cu filter_apply_pipelined); columns are independent, so every bit must equal the
    # device API's single call -- column-major (Eigen) and row-major host layouts, a ragged last chunk
    cfg = configs.CONFIGS["c2"]
    a = cfg.operator()
    da = adp.DeviceCsr(a, ctx)
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, 40, 0.5)
    for q in (256, 301):
        x = device_block(ctx, a.n_rows, q + (q % 2), seed=q)[:, :q]
        yd = adp.clenshaw_apply_device(f, da, x, 7).cpu().numpy()
        xh = x.cpu().numpy()
        yh = adp.clenshaw_apply(f, da, np.asfortranarray(xh), 7)
        assert np.array_equal(yd, yh), q
        lib = _native.lib()
        xr = np.ascontiguousarray(xh)
        yr = np.empty_like(xr)
        coeffs = f.coeff_array()
        cnt = C.c_int64(0)
        _native.check(lib.adp_filter_apply(ctx.h, da.h, coeffs.ctypes.data_as(C.c_void_p), f.k_max, f.l1, f.l2, 7,
                                           xr.ctypes.data_as(C.c_void_p), a.n_rows, q, q, 1,
                                           yr.ctypes.data_as(C.c_void_p), q, C.byref(cnt)))
        assert np.array_equal(yd, yr), q
        deg = 7  # trailing exactly-zero coefficients reduce the degree (cheb_filter.cpp:141-142)
        while deg > 0 and coeffs[deg] == 0.0:
            deg -= 1
        assert cnt.value == deg * q
