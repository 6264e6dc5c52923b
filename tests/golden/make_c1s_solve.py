"""Write tests/golden/c1s_solve.npz: the CPU solver oracle's eigenpairs on the c1s window.

The c1s configuration (config 1's 40^3 7-point operator, window of ~35 eigenvalues at 0.425 of the
range; paper_2604_00914_b200/configs.py) solved by oracle/solver_oracle.py -- the reference's solve
(proj/src/solver.cpp:119-360) restated in numpy over the oracle's C++ restatement of its kernels --
takes ~15 minutes on 8 host threads, too long to re-run inside the GPU test suite. Its eigenvalues,
residual norms and summary are stored here so tests/test_gpu_solver.py compares the GPU solve
against them on every driver run (same count, eigenvalues <= 1e-10 relative). Run in the build
container: python tests/golden/make_c1s_solve.py
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as orc  # noqa: E402
from oracle import solver_oracle  # noqa: E402
from paper_2604_00914_b200 import configs  # noqa: E402


def main():
    orc.build()
    orc.set_threads(orc.max_threads())
    configs.set_rng(orc.uniform_range, orc.gaussian_range)
    cfg = configs.CONFIGS["c1s"]
    a = cfg.operator()
    oa = orc.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    t0 = time.perf_counter()
    r = solver_oracle.solve(oa, cfg.window[0], cfg.window[1], rng_seed=0)
    secs = time.perf_counter() - t0
    res = solver_oracle.compute_residuals(oa, r.eigenvectors, r.eigenvalues)
    np.savez_compressed(os.path.join(HERE, "c1s_solve.npz"), eigenvalues=np.asarray(r.eigenvalues),
                        residuals=np.asarray(res), converged=r.converged, iterations=r.iterations,
                        e_estimate=r.e_estimate, subspace_dim=r.subspace_dim, bounds=np.asarray(r.bounds),
                        window=np.asarray(cfg.window), cpu_seconds=secs, threads=orc.max_threads())
    print(f"c1s: {len(r.eigenvalues)} eigenpairs, {r.iterations} iterations, {secs:.0f} s, max residual "
          f"{max(res):.3e}")


if __name__ == "__main__":
    main()
