"""Config 5 at FULL size (n = 4e6, ~2.16 G nonzeros > 2^31: int64 row offsets) -- GPU, opt-in (ADP_RUN_LONG=1).

The operator is generated on the device and uploaded with adp_csr_create_device. The oracle cannot
filter a 4e6 x q block, but a degree-2 Clenshaw result on row s depends only on A's rows in
L1 = {s} u cols(s) and on X's rows in L2 = L1 u cols(L1). So the full-size GPU result is checked
row by row, bitwise, against the CPU oracle run on the sub-operator that keeps A's rows L1 (columns
renumbered monotonically into L2, so every row's ascending-column accumulation order is unchanged)
and empty rows elsewhere -- for sampled rows at both ends, the middle, and random positions.
"""
import os

import numpy as np
import pytest

import paper_2604_00914_b200 as adp
from paper_2604_00914_b200 import configs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


@pytest.mark.skipif(os.environ.get("ADP_RUN_LONG") != "1", reason="full-size config 5 (~120 GB of HBM, minutes): ADP_RUN_LONG=1")
def test_c5_full_size_rows_bitwise_vs_oracle(orc):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = configs.CONFIGS["c5"]
    ctx = adp.Context(0)
    ctx.set_stream(torch.cuda.current_stream())
    rp, ci, v = cfg.device_build()
    n, nnz = rp.numel() - 1, ci.numel()
    assert nnz > 2 ** 31 and 530 < nnz / n < 550
    da = adp.DeviceCsr.from_device(n, n, rp, ci, v, ctx)
    q, degree = 128, 2
    gen = torch.Generator(device="cuda").manual_seed(11)
    x = torch.complex(torch.randn(n, q, generator=gen, dtype=torch.float64, device="cuda"),
                      torch.randn(n, q, generator=gen, dtype=torch.float64, device="cuda"))
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, 40, 0.5)
    g = orc.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, 40, 0.5)
    y = adp.clenshaw_apply_device(f, da, x, degree)
    torch.cuda.synchronize()

    rp_h = rp.cpu().numpy()
    rng = np.random.default_rng(5)
    sample = sorted({0, 1, 250, n // 2, n - 2, n - 1, *rng.integers(0, n, 4).tolist()})

    def rows_of(rows):
        idx = np.concatenate([np.arange(rp_h[r], rp_h[r + 1]) for r in rows])
        it = torch.from_numpy(idx).cuda()
        return ci[it].cpu().numpy().astype(np.int64), v[it].cpu().numpy()

    c_s, _ = rows_of(sample)
    level1 = np.union1d(sample, c_s)
    c1, v1 = rows_of(level1)
    level2 = np.union1d(level1, c1)
    m = len(level2)
    cnt = np.zeros(m, np.int64)
    pos = np.searchsorted(level2, level1)
    cnt[pos] = rp_h[level1 + 1] - rp_h[level1]
    sub_rp = np.zeros(m + 1, np.int64)
    np.cumsum(cnt, out=sub_rp[1:])
    sub = orc.Csr(m, m, sub_rp, np.searchsorted(level2, c1).astype(np.int64), v1)
    t = orc.Tiled(sub, 256, 64)
    for c0, c1_ in ((0, 2), (126, 128)):
        xs = np.asfortranarray(x[torch.from_numpy(level2).cuda(), c0:c1_].cpu().numpy())
        want = orc.clenshaw_apply(g, t, xs, degree)
        got = y[torch.tensor(sample, device="cuda"), c0:c1_].cpu().numpy()
        assert np.array_equal(got, want[np.searchsorted(level2, sample)]), (c0, c1_)
    del y, x, rp, ci, v
    da.close()
    torch.cuda.empty_cache()
