"""RunReport (proj/src/run_report.cpp) and the solve flow (proj/src/cli.cpp:152-196).

CPU: nlohmann dump(2) number/layout rules, to_json / from_json round trip,
thread-count resolution. GPU: the reference's `solve` CLI test cases
(proj/tests/test_cli.cpp:63-216) through `run_solve`.
"""
import io
import json
import math
import os

import numpy as np
import pytest

import paper_2604_00914_b200 as adp
from paper_2604_00914_b200 import report as rp


@pytest.mark.parametrize("x,want", [
    (1.0, "1.0"), (0.1, "0.1"), (-2.5, "-2.5"), (0.0, "0.0"), (-0.0, "-0.0"), (100.0, "100.0"),
    (1e-10, "1e-10"), (1.5e-5, "1.5e-05"), (0.001, "0.001"), (0.0001, "0.0001"), (1e-5, "1e-05"),
    (123456789012345.0, "123456789012345.0"), (1e15, "1e+15"), (1234567890123456.0, "1.234567890123456e+15"),
    (1.1047627945691505e-09, "1.1047627945691505e-09"), (12.34, "12.34"), (1e100, "1e+100"),
    (math.inf, "null"), (math.nan, "null"),
])
def test_format_double_nlohmann(x, want):
    assert rp.format_double(x) == want


def test_dump_layout():
    doc = {"b": [1, 2.0], "a": {"z": None, "y": True}, "e": [], "o": {}, "s": "p\"q\n"}
    want = ('{\n  "a": {\n    "y": true,\n    "z": null\n  },\n  "b": [\n    1,\n    2.0\n  ],\n  "e": [],\n'
            '  "o": {},\n  "s": "p\\"q\\n"\n}')
    assert rp.dumps(doc) == want
    assert json.loads(rp.dumps(doc)) == doc


def synthetic_report():
    hist = [adp.IterationRecord(1, 40, 12, 3, 0, 0.5, 480, 12, -1.0),
            adp.IterationRecord(2, 33, 12, 10, 10, 1e-11, 396, 12, -1.0)]
    res = adp.SolveResult(eigenvalues=np.array([11.0, 12.5, 1e-3]), eigenvectors=np.zeros((5, 3)), converged=True,
                          dense_fallback=False, iterations=2, spmv_total=1234567, avg_degree=36.5,
                          max_residual=2.5e-12, degree_history=[40, 33], history=hist,
                          bounds=adp.SpectrumBounds(-1.25, 101.0), e_estimate=9.73, subspace_dim=18,
                          timings=adp.StageTimings(setup=0.01, filter=0.2, orth=0.003, rayleigh_ritz=0.002,
                                                   residuals=0.001, other=0.0005))
    cfg = adp.SolverConfig(interval_a=10.5, interval_b=20.5, rng_seed=4, p_override=18, tile_tk=64)
    return rp.RunReport(config=cfg, threads=8, matrix_path="diag100.mtx", n=100, nnz=100, result=res)


def test_round_trip_reproduces_document():
    r = synthetic_report()
    j = json.loads(rp.dump_report(r))
    assert rp.to_json(rp.run_report_from_json(j)) == j  # test_cli.cpp:82-84
    assert rp.dump_report(rp.run_report_from_json(j)) == rp.dump_report(r)
    assert j["config"]["C"] == 1.4 and j["config"]["p_override"] == 18 and j["config"]["tile_ti"] is None
    assert j["result"]["spectrum_bounds"] == {"lambda_min": -1.25, "lambda_max": 101.0}
    assert [row["n_locked"] for row in j["iteration_table"]] == [0, 10]
    assert "device" not in j
    r.device = {"name": "NVIDIA B200", "kernel_launches": 3}
    j2 = json.loads(rp.dump_report(r))
    assert j2["device"]["kernel_launches"] == 3
    assert rp.run_report_from_json(j2).device == r.device


def test_missing_field_raises():
    j = json.loads(rp.dump_report(synthetic_report()))
    del j["result"]["e_estimate"]
    with pytest.raises(KeyError):
        rp.run_report_from_json(j)


def test_thread_count_resolution(monkeypatch):
    monkeypatch.setenv("ADAPOLY_THREADS", "3")
    assert rp.resolved_thread_count(None) == 3
    assert rp.resolved_thread_count(2) == 2
    monkeypatch.delenv("ADAPOLY_THREADS")
    assert rp.resolved_thread_count(None) >= 1


# ------------------------------------------------------------------ GPU flow ---
def write_mtx(path, a):
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr))
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{a.n_rows} {a.n_cols} {a.nnz}\n")
        for r, c, v in zip(rows, a.col_idx, a.values):
            fh.write(f"{int(r) + 1} {int(c) + 1} {float(v)!r}\n")


def diag_fixture(tmp_path, n):
    d = np.arange(1, n + 1, dtype=np.float64)
    a = adp.CsrMatrix.from_triplets(n, n, np.arange(n), np.arange(n), d)
    path = str(tmp_path / f"diag{n}.mtx")
    write_mtx(path, a)
    return path


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return adp.Context(0)


@pytest.mark.gpu
def test_solve_diag_fixture_report(gpu, tmp_path):
    out, err = io.StringIO(), io.StringIO()
    cfg = adp.SolverConfig(interval_a=10.5, interval_b=20.5, rng_seed=4)
    code, rep = adp.run_solve(diag_fixture(tmp_path, 100), cfg, ctx=gpu, output=out, err=err)
    assert code == rp.EXIT_OK
    j = json.loads(out.getvalue())
    assert j["result"]["converged"]
    ev = j["result"]["eigenvalues"]
    assert len(ev) == 10
    for i, v in enumerate(ev):
        assert v == pytest.approx(11.0 + i)
    assert j["matrix"]["n"] == 100 and j["matrix"]["nnz"] == 100
    assert rp.to_json(rp.run_report_from_json(j)) == j
    assert j["device"]["kernel_launches"] > 0


@pytest.mark.gpu
def test_solve_errors_and_iteration_cap(gpu, tmp_path):
    out, err = io.StringIO(), io.StringIO()
    code, _ = adp.run_solve("/no/such/file.mtx", adp.SolverConfig(interval_a=0, interval_b=1), ctx=gpu,
                            output=out, err=err)
    assert code == rp.EXIT_INPUT_ERROR and out.getvalue() == "" and "/no/such/file.mtx" in err.getvalue()
    # non-symmetric input
    rng = np.random.default_rng(3)
    m = (rng.random((8, 8)) < 0.4) * rng.standard_normal((8, 8))
    r, c = np.nonzero(m)
    ns = str(tmp_path / "nonsym.mtx")
    write_mtx(ns, adp.CsrMatrix.from_triplets(8, 8, r, c, m[r, c]))
    err = io.StringIO()
    code, _ = adp.run_solve(ns, adp.SolverConfig(interval_a=0, interval_b=1), ctx=gpu, err=err)
    assert code == rp.EXIT_INPUT_ERROR and "symmetric" in err.getvalue()
    # iteration cap: exit 2 with a report
    out = io.StringIO()
    cfg = adp.SolverConfig(interval_a=10.5, interval_b=20.5, rng_seed=4, max_iter=2)
    code, _ = adp.run_solve(diag_fixture(tmp_path, 100), cfg, ctx=gpu, output=out)
    assert code == rp.EXIT_NOT_CONVERGED
    assert not json.loads(out.getvalue())["result"]["converged"]


@pytest.mark.gpu
def test_solve_eigenvectors_seed_reproducibility_and_history(gpu, tmp_path):
    path = diag_fixture(tmp_path, 100)
    vec = str(tmp_path / "vecs.txt")
    report_file = str(tmp_path / "report.json")
    cfg = adp.SolverConfig(interval_a=10.5, interval_b=20.5, rng_seed=123)
    code, rep = adp.run_solve(path, cfg, ctx=gpu, threads=1, eigenvectors_path=vec, output=report_file)
    assert code == rp.EXIT_OK
    lines = open(vec).read().splitlines()
    assert lines[0] == "100 10" and len(lines) == 101
    j1 = json.load(open(report_file))
    _, rep2 = adp.run_solve(path, cfg, ctx=gpu, threads=1)
    j2 = rp.to_json(rep2)
    for j in (j1, j2):
        j.pop("timings")
    assert rp.dumps(j1) == rp.dumps(j2)  # byte-for-byte modulo timings (test_cli.cpp:177-192)
    cfg = adp.SolverConfig(interval_a=30.5, interval_b=40.5, rng_seed=8)
    _, rep3 = adp.run_solve(path, cfg, ctx=gpu)
    j3 = rp.to_json(rep3)
    assert [row["degree"] for row in j3["iteration_table"]] == j3["result"]["degree_history"]
