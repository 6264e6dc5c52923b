"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference solver.

Restates proj/src/solver.cpp:22-360 (solve, estimate_eigcount,
compute_residuals, spurious_threshold, top_up_basis), proj/src/lanczos.cpp:20-111
(estimate_spectrum_bounds) and proj/src/dense_kernels.cpp:12-101 (sym_eig,
cholesky, cholesky_qr, mgs_orthonormalize, rayleigh_ritz) on top of the pinned
C oracle (filter, Philox, CSR kernels). Eigen's dense factorizations are
replaced by LAPACK through numpy/scipy, so results agree with the reference to
rounding (not bitwise): the solver-level parity gate is a tolerance.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

from . import oracle as orc


class NotPositiveDefinite(Exception):
    pass


def sym_eig(b):  # dense_kernels.cpp:31-39
    sym = 0.5 * (b + b.T)
    w, v = np.linalg.eigh(sym)
    return w, v


def cholesky(g):  # dense_kernels.cpp:41-51 -> upper R with R^T R = G
    try:
        lower = np.linalg.cholesky(g)
    except np.linalg.LinAlgError:
        raise NotPositiveDefinite() from None
    r = lower.T
    if not np.all(np.isfinite(r)) or (g.shape[0] > 0 and r.diagonal().min() <= 0.0):
        raise NotPositiveDefinite()
    return r


def mgs_orthonormalize(x):  # dense_kernels.cpp:12-27
    n, p = x.shape
    q = np.zeros((n, p))
    kept = 0
    for j in range(p):
        v = x[:, j].copy()
        orig = np.linalg.norm(v)
        for _ in range(2):
            for i in range(kept):
                v -= (q[:, i] @ v) * q[:, i]
        nrm = np.linalg.norm(v)
        if not (nrm > orig * 1e-13) or not (nrm > 0.0):
            continue
        q[:, kept] = v / nrm
        kept += 1
    return q[:, :kept]


def cholesky_qr(x):  # dense_kernels.cpp:53-92
    p = x.shape[1]
    if p == 0:
        return x
    first_ok = False
    try:
        g = x.T @ x
        try:
            r = cholesky(g)
        except NotPositiveDefinite:
            g = g + np.eye(p) * (1e-14 * np.trace(g) / p)
            r = cholesky(g)
        for j in range(p):
            if not (r[j, j] > 1e-7 * math.sqrt(g[j, j])):
                raise NotPositiveDefinite()
        q = sla.solve_triangular(r, x.T, trans="T", lower=False).T
        first_ok = True
    except NotPositiveDefinite:
        q = mgs_orthonormalize(x)
    if not first_ok:
        return q
    try:
        r2 = cholesky(q.T @ q)
        q = sla.solve_triangular(r2, q.T, trans="T", lower=False).T
    except NotPositiveDefinite:
        q = mgs_orthonormalize(q)
    return q


def rayleigh_ritz(a: orc.Csr, q):  # dense_kernels.cpp:94-101
    aq = orc.naive_spmm(a, q)
    w, u = sym_eig(q.T @ aq)
    return w, q @ u


def compute_residuals(a, vectors, values):  # solver.cpp:94-106
    av = orc.naive_spmm(a, vectors)
    return np.linalg.norm(av - vectors * np.asarray(values)[None, :], axis=0)


def spurious_threshold(ritz, lo, hi):  # solver.cpp:81-92
    tau = math.inf
    for x in ritz:
        tau = min(tau, min(x - lo, hi - x))
    return tau


def lanczos_pass(a, steps, seed, draw_offset, spmv):  # lanczos.cpp:20-77
    n = a.n_rows
    basis = np.zeros((n, steps))
    alphas = np.zeros(steps)
    betas = np.zeros(steps)
    v = orc.gaussian_range(seed, 1, draw_offset, n)
    basis[:, 0] = v / np.linalg.norm(v)
    scale, completed, beta_res, breakdown = 0.0, 0, 0.0, False
    for j in range(steps):
        w = orc.csr_spmv(a, basis[:, j])
        spmv[0] += 1
        alphas[j] = basis[:, j] @ w
        w = w - alphas[j] * basis[:, j]
        if j > 0:
            w = w - betas[j - 1] * basis[:, j - 1]
        for _ in range(2):
            w = w - basis[:, : j + 1] @ (basis[:, : j + 1].T @ w)
        beta = np.linalg.norm(w)
        betas[j] = beta
        completed = j + 1
        scale = max(scale, abs(alphas[j]), beta)
        if beta <= scale * 1e-13:
            beta_res, breakdown = beta, True
            break
        if j + 1 < steps:
            basis[:, j + 1] = w / beta
        else:
            beta_res = beta
    tri = np.diag(alphas[:completed]) + np.diag(betas[: completed - 1], 1) + np.diag(betas[: completed - 1], -1)
    w, u = sym_eig(tri)
    r_min = beta_res * abs(u[completed - 1, 0])
    r_max = beta_res * abs(u[completed - 1, completed - 1])
    return w[0] - r_min, w[-1] + r_max, breakdown and completed < steps


def estimate_spectrum_bounds(a, steps, seed, spmv):  # lanczos.cpp:81-111
    n = a.n_rows
    eff = min(steps, n)
    lower, upper = math.inf, -math.inf
    for attempt in range(4):
        lo, hi, early = lanczos_pass(a, eff, seed, attempt * n, spmv)
        lower, upper = min(lower, lo), max(upper, hi)
        if not early:
            break
    mag = max(abs(lower), abs(upper))
    if not (upper - lower > 1e-12 * mag):
        pad = max(1e-8, np.finfo(float).eps * n * mag)
        lower, upper = lower - pad, upper + pad
    return lower, upper


def top_up_basis(q, target, seed, draw_offset):  # solver.cpp:58-77
    n = q.shape[0]
    full = np.zeros((n, target))
    full[:, : q.shape[1]] = q
    have, draw = q.shape[1], draw_offset
    while have < target:
        v = orc.gaussian_range(seed, 3, draw, n)
        draw += n
        for _ in range(2):
            v = v - full[:, :have] @ (full[:, :have].T @ v)
        nrm = np.linalg.norm(v)
        if nrm <= 1e-8:
            continue
        full[:, have] = v / nrm
        have += 1
    return full


@dataclass
class Result:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    converged: bool = False
    dense_fallback: bool = False
    iterations: int = 0
    spmv_total: int = 0
    max_residual: float = 0.0
    degree_history: list = field(default_factory=list)
    e_estimate: float = 0.0
    bounds: tuple = (0.0, 0.0)
    subspace_dim: int = 0


def solve(a: orc.Csr, interval_a, interval_b, tau_c=1e-10, tau_a=1e-3, m=0.5, c=1.4, k_multiplier=2.5, mu=1.8,
          max_iter=100, lanczos_steps=40, trace_probes=30, rng_seed=0, p_override=None, spurious_detection=True):
    """solve (solver.cpp:119-360)."""
    n = a.n_rows
    lo, hi = interval_a, interval_b
    res = Result(np.zeros(0), np.zeros((n, 0)))
    spmv = [0]
    lmin, lmax = estimate_spectrum_bounds(a, lanczos_steps, rng_seed, spmv)
    res.bounds = (lmin, lmax)
    if not (lmin <= lo and hi <= lmax):
        raise orc.ConfigError(1, "solve: target interval lies outside the estimated spectrum")
    a_norm = max(abs(lmin), abs(lmax))
    span = lmax - lmin
    l1, l2 = 2.0 / span, -(lmax + lmin) / span
    mapc = lambda x: min(max(l1 * x + l2, -1.0), 1.0)  # noqa: E731
    alpha, beta = math.acos(mapc(lo)), math.acos(mapc(hi))
    k1 = orc.initial_degree(alpha, beta, c)
    k_max = max(k1, int(math.ceil(k_multiplier * k1)))
    f = orc.build_filter(lo, hi, (lmin, lmax), k_max, m)
    tiled = orc.Tiled(a, 256, 64)
    res.e_estimate = orc.estimate_eigcount(tiled, f, trace_probes, rng_seed, spmv)
    if p_override:
        p = p_override
    else:
        if res.e_estimate < 0.5:
            res.converged = True
            res.spmv_total = spmv[0]
            return res
        e_ceil = int(math.ceil(max(res.e_estimate, 0.0)))
        p = max(int(math.ceil(mu * e_ceil)), e_ceil + 5, 10)
    res.subspace_dim = min(p, n)
    if p >= n:
        w, v = sym_eig(a.to_dense())
        sel = (w >= lo) & (w <= hi)
        res.eigenvalues, res.eigenvectors = w[sel], v[:, sel]
        r = compute_residuals(a, res.eigenvectors, res.eigenvalues)
        spmv[0] += len(res.eigenvalues)
        res.max_residual = float(r.max()) if len(r) else 0.0
        res.converged = res.dense_fallback = True
        res.spmv_total = spmv[0]
        return res
    basis = cholesky_qr(orc.fill_gaussian(n, p, rng_seed, 0))
    if basis.shape[1] < p:
        basis = top_up_basis(basis, p, rng_seed, 0)
    degree = min(k1, k_max)
    locked_vals, locked_vecs = [], []
    n_lock, n_check_prev, it, empty_streak = 0, 0, 0, 0
    hist_spmv = 0
    while it < max_iter:
        it += 1
        s = [0]
        filtered = orc.clenshaw_apply(f, tiled, basis, degree, s)
        hist_spmv += s[0]
        stacked = np.concatenate([np.array(locked_vecs).T.reshape(n, n_lock), filtered], axis=1)
        q = cholesky_qr(stacked)
        if q.shape[1] < p:
            q = top_up_basis(q, p, rng_seed, it << 32)
        ritz, basis = rayleigh_ritz(a, q[:, n_lock:])
        inside = [j for j in range(len(ritz)) if lo <= ritz[j] <= hi]
        e_i = len(inside)
        res.degree_history.append(degree)
        res.iterations = it
        if e_i == 0:
            empty_streak += 1
            if it > 3 and empty_streak >= 10:
                res.converged = True
                break
            continue
        empty_streak = 0
        fi = orc.ChebFilter(f.interval_a, f.interval_b, f.alpha, f.beta, f.k_max, f.m, f.l1, f.l2, f.lambda_min,
                            f.lambda_max, f.coeffs, f.active_degree)
        next_degree = orc.adaptive_degree(fi, ritz, e_i, tau_a)
        vals_in = ritz[inside]
        resid = compute_residuals(a, basis[:, inside], vals_in)
        hist_spmv += e_i
        tau_s = spurious_threshold(vals_in, lo, hi)
        test_set = list(range(e_i))
        if spurious_detection and tau_s > 0.0:
            checked = [cc for cc in range(e_i) if resid[cc] < tau_s]
            n_check = len(checked) + n_lock
            if n_check > 0 and n_check == n_check_prev:
                test_set = checked
            n_check_prev = n_check
        lock = set()
        n_unconv = 0
        for cc in test_set:
            if resid[cc] < tau_c * a_norm:
                j = inside[cc]
                lock.add(j)
                locked_vals.append(ritz[j])
                locked_vecs.append(basis[:, j].copy())
            else:
                n_unconv += 1
        n_lock += len(lock)
        if lock:
            basis = basis[:, [j for j in range(basis.shape[1]) if j not in lock]]
        degree = next_degree
        if n_unconv == 0:
            res.converged = True
            break
    order = np.argsort(np.array(locked_vals), kind="stable") if locked_vals else np.zeros(0, int)
    res.eigenvalues = np.array(locked_vals)[order] if locked_vals else np.zeros(0)
    res.eigenvectors = np.array(locked_vecs).T[:, order] if locked_vals else np.zeros((n, 0))
    if n_lock:
        r = compute_residuals(a, res.eigenvectors, res.eigenvalues)
        spmv[0] += n_lock
        res.max_residual = float(r.max())
    res.spmv_total = spmv[0] + hist_spmv
    return res
