"""The row-sharded solve (paper_2604_00914_b200/sharded.py) on the CPU: gloo ranks, numpy backend.

The same solve loop the GPU runs (sharded.ShardedSolver: the reference's solve, solver.cpp:119-360,
with every n-sized reduction allreduced) over world = 1, 2, 3 ranks, the filter and SpMM through the
row-partitioned DistributedFilter with the numpy step backend. Bar (BASELINE.json north_star):
eigenvalues in [a, b] agree with the single process and with the CPU solver oracle (the reference's
solve restated) to <= 1e-10 relative, with the same count and all residuals under the tolerance.
Complex Hermitian (config 3's structure) runs the same loop with complex128 blocks.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind):
    sys.path.insert(0, ROOT)
    from paper_2604_00914_b200 import configs

    if kind == "lap":  # 10^3 7-point + U[0,1): a window of ~10 eigenvalues at 0.425 of the range
        return configs.laplacian7_potential(10, 0.0, 1.0, seed=2), (5.50, 5.62)
    if kind == "27pt":
        return configs.dft_like_27pt(8, n_centres=3, seed=1), (1.0, 1.25)
    return configs.peierls_lattice(14, phi=1.0 / 7.0), (-0.35, -0.2)  # complex Hermitian


def _worker(rank, world, port, kind, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from dist_numpy_backend import NumpyStepBackend
    from paper_2604_00914_b200.distributed import DistributedFilter
    from paper_2604_00914_b200.sharded import NumpyOps, ShardedSolver, ShardSparse, TorchComm
    from paper_2604_00914_b200.solver import SolverConfig

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, (lo, hi) = _problem(kind)
    df = DistributedFilter(a, NumpyStepBackend(), rank, world)
    solver = ShardedSolver(a.n_rows, a.is_complex, NumpyOps(a.is_complex), ShardSparse(df), TorchComm())
    r = solver.solve(SolverConfig(interval_a=lo, interval_b=hi, rng_seed=3))
    np.savez(f"{out_path}.{rank}.npz", values=r.eigenvalues, vectors=np.asarray(r.eigenvectors),
             converged=r.converged, max_residual=r.max_residual, e_estimate=r.e_estimate, p=r.subspace_dim,
             bounds=np.array([r.bounds.lambda_min, r.bounds.lambda_max]))
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, kind, world):
    import torch.multiprocessing as mp

    out = str(tmp_path / f"{kind}{world}")
    mp.start_processes(_worker, args=(world, _free_port(), kind, out), nprocs=world, join=True, start_method="spawn")
    return [np.load(f"{out}.{r}.npz") for r in range(world)]


@pytest.mark.parametrize("kind", ["lap", "27pt", "herm"])
def test_sharded_solve_matches_single_process_and_oracle(tmp_path, orc, kind):
    a, (lo, hi) = _problem(kind)
    one = _run(tmp_path, kind, 1)[0]
    assert bool(one["converged"]) and len(one["values"]) >= 4
    a_norm = np.max(np.abs(one["bounds"]))
    assert float(one["max_residual"]) <= 1e-10 * a_norm * 1.0001
    # every eigenvalue of the dense spectrum inside [a, b] is found (same count)
    dense = np.linalg.eigvalsh(a.to_dense())
    want = dense[(dense >= lo) & (dense <= hi)]
    assert len(one["values"]) == len(want)
    assert np.max(np.abs(one["values"] - want) / np.abs(want)) <= 1e-10
    if kind != "herm":  # the CPU solver oracle (the reference's solve restated, real symmetric)
        from oracle import solver_oracle

        ref = solver_oracle.solve(orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), lo, hi, rng_seed=3)
        assert len(ref.eigenvalues) == len(one["values"])
        assert np.max(np.abs(np.sort(ref.eigenvalues) - one["values"]) / np.abs(one["values"])) <= 1e-10
    for world in ((2, 3) if kind == "lap" else (3,)):
        parts = _run(tmp_path, kind, world)
        vals = parts[0]["values"]
        for p in parts[1:]:
            assert np.array_equal(p["values"], vals)  # replicated host logic: every rank agrees
        assert len(vals) == len(one["values"])
        assert np.max(np.abs(vals - one["values"]) / np.abs(one["values"])) <= 1e-10
        vecs = np.concatenate([p["vectors"] for p in parts])  # rows of the partition, stacked
        assert vecs.shape == (a.n_rows, len(vals))
        res = np.linalg.norm(a.to_dense() @ vecs - vecs * vals[None, :], axis=0)
        assert np.max(res) <= 1e-10 * a_norm * 1.0001
        assert np.allclose(vecs.conj().T @ vecs, np.eye(len(vals)), atol=1e-12)
