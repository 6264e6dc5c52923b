"""The row-sharded / complex solve (paper_2604_00914_b200/sharded.py) on the GPU.

* world 1, real: ShardedSolver with the device filter and torch (cuBLAS / cuSOLVER) dense steps equals
  the C++ device solver (adp.solve) to <= 1e-10 relative, same count;
* emulated ranks: 2 and 3 ranks as threads on ONE GPU (B200_PROFILING.md: no kernel waits on another
  rank's kernel -- halo rows move through a host mailbox, allreduces through a host barrier), each
  rank's filter the product's row-partitioned DistributedFilter over the CUDA step backend; eigenvalues
  equal the single-process solve to <= 1e-10 with the same count; real and complex Hermitian.
"""
import threading

import numpy as np
import pytest

import paper_2604_00914_b200 as adp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


class ThreadComm:
    """allreduce(sum) across emulated ranks (threads): host copies, one fixed summation order."""

    def __init__(self, shared, rank, world):
        self.shared, self.rank, self.world = shared, rank, world

    def allreduce(self, x):
        sh = self.shared
        host = x.detach().cpu().numpy().copy() if hasattr(x, "detach") else np.array(x)
        with sh["cv"]:
            gen = sh["gen"]
            sh["slots"][self.rank] = host
            sh["count"] += 1
            if sh["count"] == self.world:
                sh["result"] = sum(sh["slots"][k] for k in range(self.world))
                sh["count"] = 0
                sh["gen"] += 1
                sh["cv"].notify_all()
            else:
                while sh["gen"] == gen:
                    sh["cv"].wait(timeout=120)
            out = sh["result"].copy()
        return torch.as_tensor(out, device=x.device) if hasattr(x, "device") else out


def _problem(kind):
    from paper_2604_00914_b200 import configs

    if kind == "lap":
        return configs.laplacian7_potential(12, 0.0, 1.0, seed=2), (5.50, 5.60)
    return configs.peierls_lattice(16, phi=1.0 / 8.0, seed=1), (-0.3, -0.15)


def test_sharded_world1_equals_cpp_solver():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_00914_b200.sharded import solve_sharded, LocalComm

    a, (lo, hi) = _problem("lap")
    cfg = adp.SolverConfig(interval_a=lo, interval_b=hi, rng_seed=3)
    ctx = adp.Context(0)
    want = adp.solve(adp.DeviceCsr(a, ctx), cfg)
    got = solve_sharded(a, cfg, comm=LocalComm(), ctx=ctx)
    assert got.converged and want.converged
    assert len(got.eigenvalues) == len(want.eigenvalues) > 3
    assert np.max(np.abs(got.eigenvalues - want.eigenvalues) / np.abs(want.eigenvalues)) <= 1e-10
    scale = max(abs(want.bounds.lambda_min), abs(want.bounds.lambda_max))
    assert got.max_residual <= 1e-10 * scale * 1.0001
    ctx.close()


@pytest.mark.parametrize("kind,world", [("lap", 2), ("lap", 3), ("herm", 2)])
def test_sharded_emulated_ranks_match_single(kind, world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_distributed import Mailbox, make_backend

    from paper_2604_00914_b200.distributed import DistributedFilter
    from paper_2604_00914_b200.sharded import LocalComm, ShardedSolver, ShardSparse, TorchOps, solve_sharded

    a, (lo, hi) = _problem(kind)
    cfg = adp.SolverConfig(interval_a=lo, interval_b=hi, rng_seed=5)
    one = solve_sharded(a, cfg, comm=LocalComm())
    assert one.converged and len(one.eigenvalues) > 3
    mailbox = Mailbox()
    shared = {"cv": threading.Condition(), "gen": 0, "count": 0, "slots": {}, "result": None}
    results, errors = [None] * world, []

    def body(rank):
        try:
            be = make_backend(mailbox, rank)
            with torch.cuda.stream(be.stream):
                df = DistributedFilter(a, be, rank, world)
                s = ShardedSolver(a.n_rows, a.is_complex, TorchOps(a.is_complex), ShardSparse(df),
                                  ThreadComm(shared, rank, world))
                results[rank] = s.solve(cfg)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errors:
        raise errors[0]
    for r in results:
        assert r.converged and len(r.eigenvalues) == len(one.eigenvalues)
        assert np.max(np.abs(r.eigenvalues - one.eigenvalues) / np.abs(one.eigenvalues)) <= 1e-10
    vecs = np.concatenate([r.eigenvectors.cpu().numpy() for r in results])
    res = np.linalg.norm(a.to_dense() @ vecs - vecs * one.eigenvalues[None, :], axis=0)
    scale = max(abs(one.bounds.lambda_min), abs(one.bounds.lambda_max))
    assert np.max(res) <= 1e-10 * scale * 1.0001
