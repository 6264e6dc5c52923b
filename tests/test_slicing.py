"""Spectrum-slicing driver (paper_2604_00914_b200/slicing.py).

CPU: slice cutting, edge ownership and the multi-rank merge with a stand-in
solver (gloo, world_size 2: every rank solves its slices, the pairs are
exchanged once). GPU: slices of a diagonal spectrum solved on the device
reproduce the single-interval solve.
"""
import os
import pickle
import socket
import sys

import numpy as np
import pytest

import paper_2604_00914_b200 as adp
from paper_2604_00914_b200 import slicing

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPECTRUM = np.array([0.5, 1.0, 2.0, 2.5, 3.0, 3.25, 4.0, 5.0, 6.0, 7.5])  # 2.0, 4.0, 6.0 fall on slice edges


class FakeResult:
    def __init__(self, lo, hi):
        sel = np.nonzero((SPECTRUM >= lo) & (SPECTRUM <= hi))[0]  # closed interval, like the solver
        self.eigenvalues = SPECTRUM[sel]
        self.eigenvectors = np.eye(len(SPECTRUM))[:, sel]
        self.converged = True
        self.iterations = 1
        self.spmv_total = 10 * len(sel)


def fake_solve(_dev, cfg):
    return FakeResult(cfg.interval_a, cfg.interval_b)


def test_slice_interval():
    s = adp.slice_interval(0.0, 6.0, 3)
    assert s == [(0.0, 2.0), (2.0, 4.0), (4.0, 6.0)]
    with pytest.raises(adp.ConfigError):
        adp.slice_interval(1.0, 1.0, 2)
    with pytest.raises(adp.ConfigError):
        adp.slice_interval(0.0, 1.0, 0)


def test_repeated_eigenvalue_on_an_edge_keeps_its_multiplicity():
    global SPECTRUM
    saved = SPECTRUM
    SPECTRUM = np.array([1.0, 2.0, 2.0, 3.0])  # a double eigenvalue exactly on the edge 2.0
    try:
        r = adp.solve_sliced(None, adp.SolverConfig(interval_a=0.0, interval_b=4.0), n_slices=2, solve_fn=fake_solve)
        assert np.array_equal(r.eigenvalues, [1.0, 2.0, 2.0, 3.0])
    finally:
        SPECTRUM = saved


def test_single_process_merge_owns_each_edge_once():
    cfg = adp.SolverConfig(interval_a=0.0, interval_b=6.0)
    r = adp.solve_sliced(None, cfg, n_slices=3, solve_fn=fake_solve)
    want = SPECTRUM[(SPECTRUM >= 0.0) & (SPECTRUM <= 6.0)]
    assert np.array_equal(r.eigenvalues, want)
    assert np.array_equal(r.eigenvectors, np.eye(len(SPECTRUM))[:, np.searchsorted(SPECTRUM, want)])
    assert r.converged and sum(s.n_eigs for s in r.slices) == len(want)
    assert r.spmv_total == sum(s.spmv_total for s in r.slices)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from paper_2604_00914_b200 import SolverConfig, solve_sliced
    from test_slicing import fake_solve

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = solve_sliced(None, SolverConfig(interval_a=0.0, interval_b=7.5), n_slices=5, solve_fn=fake_solve)
    with open(f"{out_path}.{rank}.pkl", "wb") as fh:
        pickle.dump((r.eigenvalues, r.eigenvectors, [(s.lo, s.hi, s.rank, s.n_eigs) for s in r.slices]), fh)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_slices_gloo(tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "r")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    res = [pickle.load(open(f"{out}.{r}.pkl", "rb")) for r in range(2)]
    for vals, vecs, slices in res:
        assert np.array_equal(vals, SPECTRUM)  # [0, 7.5] holds all ten, each once
        assert np.array_equal(vecs, np.eye(len(SPECTRUM)))
        assert [s[2] for s in slices] == [0, 1, 0, 1, 0]  # rank r solved slices r, r + 2, ...
        assert sum(s[3] for s in slices) == len(SPECTRUM)  # overlap duplicates dropped
    assert res[0][2] == res[1][2]


@pytest.mark.gpu
def test_sliced_device_solve_matches_single_interval():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = adp.Context(0)
    n = 100
    a = adp.CsrMatrix.from_triplets(n, n, np.arange(n), np.arange(n), np.arange(1, n + 1, dtype=np.float64))
    da = adp.DeviceCsr(a, ctx)
    cfg = adp.SolverConfig(interval_a=10.5, interval_b=40.5, rng_seed=4)
    whole = adp.solve(da, cfg)
    for slices in (adp.slice_interval(10.5, 40.5, 3), adp.balanced_slices(da, 10.5, 40.5, 3, cfg)):
        r = adp.solve_sliced(da, cfg, slices=slices)
        assert r.converged and len(r.eigenvalues) == 30
        np.testing.assert_allclose(r.eigenvalues, np.arange(11.0, 41.0), rtol=1e-10)
        np.testing.assert_allclose(r.eigenvalues, whole.eigenvalues, rtol=1e-10)
        # eigenvector j is +-e_(10+j)
        assert np.allclose(np.abs(r.eigenvectors[10:40, :]), np.eye(30), atol=1e-8)
    counts = [s.n_eigs for s in adp.solve_sliced(da, cfg, slices=adp.balanced_slices(da, 10.5, 40.5, 3, cfg)).slices]
    assert min(counts) >= 7 and max(counts) <= 13  # balanced by the (noisy, 30-probe) trace estimate
    ctx.close()
