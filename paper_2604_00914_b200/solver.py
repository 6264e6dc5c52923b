"""Solver-level API: SolverConfig / solve and the device subsystems.

Mirrors proj/include/adapoly/solver.hpp (SolverConfig :14-32, IterationRecord
:49-59, StageTimings :61-68, SolveResult :70-85, solve :106), lanczos.hpp
(estimate_spectrum_bounds) and dense_kernels.hpp (cholesky_qr, rayleigh_ritz)
over the C-ABI. All n-sized work runs on the GPU (libadp_b200.so).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._native import check, lib
from .filter import ChebFilter, SpectrumBounds
from .operator import DeviceCsr


class CSolverConfig(C.Structure):
    _fields_ = [("interval_a", C.c_double), ("interval_b", C.c_double), ("tau_c", C.c_double),
                ("tau_a", C.c_double), ("m", C.c_double), ("c", C.c_double), ("k_multiplier", C.c_double),
                ("mu", C.c_double), ("max_iter", C.c_int64), ("lanczos_steps", C.c_int64),
                ("trace_probes", C.c_int64), ("rng_seed", C.c_uint64), ("p_override", C.c_int64),
                ("spurious_detection", C.c_int32), ("collect_diagnostics", C.c_int32)]


class CIterationRecord(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("degree", C.c_int32), ("active_width", C.c_int64),
                ("e_in_interval", C.c_int64), ("n_locked_total", C.c_int64), ("max_residual", C.c_double),
                ("spmv_filter", C.c_int64), ("spmv_residual", C.c_int64), ("orth_error", C.c_double)]


class CStageTimings(C.Structure):
    _fields_ = [("setup", C.c_double), ("filter", C.c_double), ("orth", C.c_double),
                ("rayleigh_ritz", C.c_double), ("residuals", C.c_double), ("other", C.c_double)]


class CSolveSummary(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_eigs", C.c_int64), ("iterations", C.c_int64), ("spmv_total", C.c_int64),
                ("subspace_dim", C.c_int64), ("n_history", C.c_int64), ("converged", C.c_int32),
                ("dense_fallback", C.c_int32), ("avg_degree", C.c_double), ("max_residual", C.c_double),
                ("e_estimate", C.c_double), ("lambda_min", C.c_double), ("lambda_max", C.c_double),
                ("timings", CStageTimings)]


@dataclass
class SolverConfig:
    """SolverConfig (solver.hpp:14-32) with the reference defaults."""

    interval_a: float = 0.0
    interval_b: float = 0.0
    tau_c: float = 1e-10
    tau_a: float = 1e-3
    m: float = 0.5
    c: float = 1.4
    k_multiplier: float = 2.5
    mu: float = 1.8
    max_iter: int = 100
    lanczos_steps: int = 40
    trace_probes: int = 30
    rng_seed: int = 0
    p_override: int | None = None
    spurious_detection: bool = True
    collect_diagnostics: bool = False
    # The reference's CPU tiling knobs (solver.hpp:28-29, csr_to_tiled T_i / T_k). The GPU keeps CSR
    # and does not use them; they are accepted so configs and RunReports round-trip unchanged.
    tile_ti: int | None = None
    tile_tk: int | None = None

    def to_c(self) -> CSolverConfig:
        return CSolverConfig(self.interval_a, self.interval_b, self.tau_c, self.tau_a, self.m, self.c,
                             self.k_multiplier, self.mu, self.max_iter, self.lanczos_steps, self.trace_probes,
                             self.rng_seed, self.p_override or 0, int(self.spurious_detection),
                             int(self.collect_diagnostics))


@dataclass
class IterationRecord:
    iteration: int
    degree: int
    active_width: int
    e_in_interval: int
    n_locked_total: int
    max_residual: float
    spmv_filter: int
    spmv_residual: int
    orth_error: float


@dataclass
class StageTimings:
    setup: float = 0.0
    filter: float = 0.0
    orth: float = 0.0
    rayleigh_ritz: float = 0.0
    residuals: float = 0.0
    other: float = 0.0


@dataclass
class SolveResult:
    """SolveResult (solver.hpp:70-85)."""

    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    converged: bool
    dense_fallback: bool
    iterations: int
    spmv_total: int
    avg_degree: float
    max_residual: float
    degree_history: list
    history: list
    bounds: SpectrumBounds
    e_estimate: float
    subspace_dim: int
    timings: StageTimings = field(default_factory=StageTimings)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def solve(a: DeviceCsr, config: SolverConfig) -> SolveResult:
    """solve (solver.hpp:106, solver.cpp:119-360) on the GPU."""
    L = lib()
    h = C.c_void_p()
    cfg = config.to_c()
    check(L.adp_solve(a.ctx.h, a.h, C.byref(cfg), C.byref(h)))
    try:
        s = CSolveSummary()
        check(L.adp_solve_summary_get(h, C.byref(s)))
        vals = np.empty(s.n_eigs)
        vecs = np.empty((s.n, s.n_eigs), order="F")
        check(L.adp_solve_eigenpairs(h, _ptr(vals), _ptr(vecs), max(s.n, 1)))
        recs = (CIterationRecord * max(s.n_history, 1))()
        degs = np.empty(max(s.n_history, 1), np.int32)
        check(L.adp_solve_history(h, recs, _ptr(degs)))
    finally:
        L.adp_solve_result_destroy(h)
    hist = [IterationRecord(r.iteration, r.degree, r.active_width, r.e_in_interval, r.n_locked_total,
                            r.max_residual, r.spmv_filter, r.spmv_residual, r.orth_error)
            for r in list(recs)[: s.n_history]]
    t = s.timings
    return SolveResult(vals, vecs, bool(s.converged), bool(s.dense_fallback), s.iterations, s.spmv_total,
                       s.avg_degree, s.max_residual, [int(d) for d in degs[: s.n_history]], hist,
                       SpectrumBounds(s.lambda_min, s.lambda_max), s.e_estimate, s.subspace_dim,
                       StageTimings(t.setup, t.filter, t.orth, t.rayleigh_ritz, t.residuals, t.other))


def estimate_spectrum_bounds(a: DeviceCsr, steps: int, seed: int, spmv_count: list | None = None) -> SpectrumBounds:
    """estimate_spectrum_bounds (lanczos.hpp:24-26): Lanczos on the device."""
    lo, hi = C.c_double(), C.c_double()
    cnt = C.c_int64(spmv_count[0] if spmv_count else 0)
    check(lib().adp_lanczos_bounds(a.ctx.h, a.h, int(steps), int(seed), C.byref(lo), C.byref(hi), C.byref(cnt)))
    if spmv_count is not None:
        spmv_count[0] = cnt.value
    return SpectrumBounds(lo.value, hi.value)


def estimate_eigcount(a: DeviceCsr, f: ChebFilter, probes: int, seed: int, spmv_count: list | None = None) -> float:
    """estimate_eigcount (solver.hpp:102-103)."""
    out = C.c_double()
    cnt = C.c_int64(spmv_count[0] if spmv_count else 0)
    coeffs = f.coeff_array()
    check(lib().adp_estimate_eigcount(a.ctx.h, a.h, _ptr(coeffs), f.k_max, f.l1, f.l2, int(probes), int(seed),
                                      C.byref(out), C.byref(cnt)))
    if spmv_count is not None:
        spmv_count[0] = cnt.value
    return out.value


def spurious_threshold(ritz_in_interval, a: float, b: float) -> float:
    """spurious_threshold (solver.hpp:92)."""
    r = np.ascontiguousarray(ritz_in_interval, np.float64)
    out = C.c_double()
    check(lib().adp_spurious_threshold(_ptr(r), len(r), a, b, C.byref(out)))
    return out.value


def cholesky_qr_device(x):
    """cholesky_qr (dense_kernels.hpp:22) in place on a torch CUDA row-major (n, p) tensor; returns kept columns."""
    import torch

    kept = C.c_int64()
    ctx = _ctx_for(x)
    ctx.set_stream(torch.cuda.current_stream(x.device))
    check(lib().adp_cholesky_qr_device(ctx.h, C.c_void_p(x.data_ptr()), x.shape[0], x.shape[1], x.stride(0),
                                       C.byref(kept)))
    return kept.value


def rayleigh_ritz_device(a: DeviceCsr, q):
    """rayleigh_ritz (dense_kernels.hpp:31): returns (theta ascending, V = Q U as a new tensor)."""
    import torch

    qc = q.shape[1]
    theta = np.empty(qc)
    v = torch.empty_like(q)
    a.ctx.set_stream(torch.cuda.current_stream(q.device))
    check(lib().adp_rayleigh_ritz_device(a.ctx.h, a.h, C.c_void_p(q.data_ptr()), q.stride(0), qc, _ptr(theta),
                                         C.c_void_p(v.data_ptr()), v.stride(0)))
    return theta, v


def compute_residuals_device(a: DeviceCsr, v, values) -> np.ndarray:
    """compute_residuals (solver.hpp:96-98) for a torch CUDA row-major (n, e) block."""
    import torch

    lam = np.ascontiguousarray(values, np.float64)
    out = np.empty(len(lam))
    a.ctx.set_stream(torch.cuda.current_stream(v.device))
    check(lib().adp_residual_norms_device(a.ctx.h, a.h, C.c_void_p(v.data_ptr()), v.stride(0), v.shape[1],
                                          _ptr(lam), _ptr(out)))
    return out


def _ctx_for(t):
    from .operator import default_context

    return default_context(t.device.index or 0)
