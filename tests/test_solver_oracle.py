"""Pin the CPU solver restatement (oracle/solver_oracle.py) to the reference's own solver tests
(proj/tests/test_eigensolver.cpp) -- CPU only."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def so(orc):
    from oracle import solver_oracle

    return solver_oracle


def iota(orc, n):
    return orc.make_diag(np.arange(1, n + 1, dtype=np.float64))


def test_oracle_solve_diagonal_slice(orc, so):  # test_eigensolver.cpp:168-192
    res = so.solve(iota(orc, 100), 10.5, 20.5, rng_seed=7)
    assert res.converged and len(res.eigenvalues) == 10
    assert np.allclose(res.eigenvalues, np.arange(11, 21), rtol=1e-9, atol=0)
    assert res.max_residual <= 1e-10 * 100 * 1.01


def test_oracle_solve_empty_and_dense(orc, so):  # :194-236
    res = so.solve(iota(orc, 60), 30.3, 30.7, rng_seed=3)
    assert res.converged and len(res.eigenvalues) == 0 and res.iterations == 0
    res = so.solve(iota(orc, 60), 30.3, 30.7, rng_seed=3, p_override=8)
    assert res.converged and len(res.eigenvalues) == 0 and 10 <= res.iterations <= 15
    a = orc.random_symmetric(30, 0.3, 55)
    sp = np.linalg.eigvalsh(a.to_dense())
    res = so.solve(a, sp[5] - 1e-9, sp[24] + 1e-9, rng_seed=1, p_override=30)
    assert res.dense_fallback and len(res.eigenvalues) == 20
    assert np.allclose(res.eigenvalues, sp[5:25], rtol=1e-12, atol=0)


def test_oracle_solve_locks(orc, so):  # :314-336
    a = orc.random_symmetric(150, 0.06, 91)
    sp = np.linalg.eigvalsh(a.to_dense())
    res = so.solve(a, 0.5 * (sp[59] + sp[60]), 0.5 * (sp[74] + sp[75]), rng_seed=19)
    a_norm = max(abs(res.bounds[0]), abs(res.bounds[1]))
    assert res.converged and len(res.eigenvalues) == 15
    assert np.all(np.abs(res.eigenvalues - sp[60:75]) <= 1e-8 * a_norm)


def test_oracle_bounds_enclose(orc, so):  # :59-70 (20 seeds)
    a = orc.random_symmetric(300, 0.05, 77)
    sp = np.linalg.eigvalsh(a.to_dense())
    ok = 0
    for seed in range(20):
        lo, hi = so.estimate_spectrum_bounds(a, 40, seed, [0])
        ok += lo <= sp[0] and hi >= sp[-1]
    assert ok >= 19
