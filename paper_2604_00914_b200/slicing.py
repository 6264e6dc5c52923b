"""Spectrum slicing: one target interval split into slices solved independently.

Config 5 is "replicas only": its random off-band entries make a
row partition an all-to-all, so every GPU holds the whole operator and solves
its own window of the spectrum (the paper's parallel-in-spectrum use of the
filter). This module is that driver:

* `slice_interval` cuts [a, b] into equal-width slices; `balanced_slices`
  re-cuts them so every slice holds about the same number of eigenvalues, from
  the device trace estimate (estimate_eigcount, solver.cpp:108-117) on a
  finer grid -- solve cost grows with the slice's subspace size;
* `solve_sliced` runs `solve` once per slice -- under torch.distributed every
  rank takes slices rank, rank + W, ... on its own GPU (no data-path
  collective; results are exchanged once at the end with all_gather_object),
  else all slices run on the given context in turn -- and merges the pairs.
  Each slice is SOLVED on its interval widened by `overlap` x its width at
  the interior edges -- an eigenvalue on (or next to) an edge sits where the
  step filter is 1/2 and may never converge there, but it is then well inside
  a neighbour's solve interval -- and pairs found twice in an overlap are
  kept once (matched one to one, so multiplicities survive).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._native import ConfigError


@dataclass
class SliceOutcome:
    lo: float
    hi: float
    converged: bool
    n_eigs: int
    iterations: int
    spmv_total: int
    seconds: float
    rank: int = 0


@dataclass
class SlicedResult:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    converged: bool
    spmv_total: int
    slices: list = field(default_factory=list)


def slice_interval(a: float, b: float, n_slices: int) -> list[tuple[float, float]]:
    """Equal-width slices of [a, b]; edges are exact (the last slice ends at b)."""
    if not a < b:
        raise ConfigError("slice_interval: need a < b")
    if n_slices < 1:
        raise ConfigError("slice_interval: need at least one slice")
    edges = [a + (b - a) * i / n_slices for i in range(n_slices)] + [b]
    return [(edges[i], edges[i + 1]) for i in range(n_slices)]


def balanced_slices(dev_csr, a: float, b: float, n_slices: int, config=None, grid: int = 4) -> list[tuple[float, float]]:
    """Slices of [a, b] holding about equal eigenvalue counts (estimated on n_slices * grid cells)."""
    import math

    from .filter import build_filter, initial_degree
    from .solver import SolverConfig, estimate_eigcount, estimate_spectrum_bounds

    cfg = config or SolverConfig()
    cells = slice_interval(a, b, n_slices * grid)
    bounds = estimate_spectrum_bounds(dev_csr, cfg.lanczos_steps, cfg.rng_seed)

    def count(lo, hi):  # the solver's own setup estimate for the cell (solver.cpp:129-156)
        span = bounds.lambda_max - bounds.lambda_min
        l1, l2 = 2.0 / span, -(bounds.lambda_max + bounds.lambda_min) / span
        alpha = math.acos(min(max(l1 * lo + l2, -1.0), 1.0))
        beta = math.acos(min(max(l1 * hi + l2, -1.0), 1.0))
        k1 = initial_degree(alpha, beta, cfg.c)
        f = build_filter(lo, hi, bounds, max(k1, int(math.ceil(cfg.k_multiplier * k1))), cfg.m)
        return max(estimate_eigcount(dev_csr, f, cfg.trace_probes, cfg.rng_seed), 0.0)

    counts = np.array([count(lo, hi) for lo, hi in cells])
    if counts.sum() <= 0:
        return slice_interval(a, b, n_slices)
    cum = np.concatenate([[0.0], np.cumsum(counts)])
    edges = [a]
    for i in range(1, n_slices):
        target = cum[-1] * i / n_slices
        j = min(max(int(np.searchsorted(cum, target)), 1), len(cells))  # cell j-1 holds the target count
        c_lo, c_hi = cells[j - 1]
        frac = (target - cum[j - 1]) / counts[j - 1] if counts[j - 1] > 0 else 1.0
        e = c_lo + min(max(frac, 0.0), 1.0) * (c_hi - c_lo)  # uniform density inside the cell
        edges.append(max(e, edges[-1]))
    edges.append(b)
    out = [(edges[i], edges[i + 1]) for i in range(n_slices)]
    return [s for s in out if s[1] > s[0]] or [(a, b)]


def solve_sliced(dev_csr, config, n_slices: int | None = None, slices=None, group=None, solve_fn=None,
                 overlap: float = 0.01, rtol: float = 1e-8) -> SlicedResult:
    """Solve config.interval_a..interval_b slice by slice and merge (see the module docstring).

    ``solve_fn(dev_csr, cfg) -> SolveResult`` defaults to the GPU `solve` (to the native complex
    `solve_hermitian` when ``dev_csr`` is complex -- a host CsrMatrix or a device-generated DeviceCsr:
    config 5's slices); tests inject a stand-in.
    Pairs found by two neighbouring slices inside their overlap (values within rtol x scale) are
    kept once; genuinely repeated eigenvalues are matched one to one, so multiplicities survive.
    """
    import dataclasses
    import time

    from .solver import solve

    if solve_fn is None:
        if getattr(dev_csr, "is_complex", False):  # host CsrMatrix or device-generated DeviceCsr (config 5)
            from .hermitian import solve_hermitian

            solve_fn = solve_hermitian  # native complex128 solve on this rank's current GPU
        else:
            solve_fn = solve
    a, b = float(config.interval_a), float(config.interval_b)
    if slices is None:
        slices = slice_interval(a, b, n_slices or 1)
    slices = [(float(lo), float(hi)) for lo, hi in slices]
    last = len(slices) - 1
    pads = [overlap * (hi - lo) for lo, hi in slices]
    rank, world = 0, 1
    dist = None
    try:
        import torch.distributed as _dist

        if _dist.is_available() and _dist.is_initialized():
            dist = _dist
            rank, world = dist.get_rank(group), dist.get_world_size(group)
    except ImportError:
        pass
    mine = []
    for i in range(rank, len(slices), world):
        lo, hi = slices[i]
        s_lo = lo - pads[i] if i > 0 else lo
        s_hi = hi + pads[i] if i < last else hi
        t0 = time.perf_counter()
        r = solve_fn(dev_csr, dataclasses.replace(config, interval_a=s_lo, interval_b=s_hi))
        vals = np.asarray(r.eigenvalues, np.float64)
        vecs = np.asarray(r.eigenvectors)
        if not (vecs.ndim == 2 and vecs.shape[1] == len(vals)):
            vecs = np.zeros((0, len(vals)))
        mine.append((i, vals, vecs, SliceOutcome(lo, hi, bool(r.converged), 0, int(r.iterations), int(r.spmv_total),
                                                 time.perf_counter() - t0, rank)))
    if dist is not None and world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, mine, group=group)
        parts = [p for g in gathered for p in g]
    else:
        parts = mine
    parts.sort(key=lambda p: p[0])
    scale = max(abs(a), abs(b), b - a, 1e-300)
    tol = rtol * scale
    kept_vals, kept_vecs, kept_from = [], [], []
    for i, vals, vecs, outcome in parts:
        lo, hi = slices[i]
        # candidates of slice i-1 that lie in the overlap around this slice's left edge
        zone_lo, zone_hi = lo - pads[i - 1] - tol if i > 0 else -np.inf, lo + pads[i] + tol if i > 0 else -np.inf
        prev = [j for j, (v, s) in enumerate(zip(kept_vals, kept_from)) if s == i - 1 and zone_lo <= v <= zone_hi]
        used = set()
        for k in np.argsort(vals, kind="stable"):
            v = float(vals[k])
            if not (a <= v <= b):
                continue
            if zone_lo <= v <= zone_hi:
                match = next((j for j in prev if j not in used and abs(kept_vals[j] - v) <= tol), None)
                if match is not None:
                    used.add(match)
                    continue
            kept_vals.append(v)
            kept_vecs.append(vecs[:, k] if vecs.shape[0] else None)
            kept_from.append(i)
        outcome.n_eigs = sum(1 for s in kept_from if s == i)
    order = np.argsort(np.array(kept_vals), kind="stable")
    vals = np.array(kept_vals, np.float64)[order] if kept_vals else np.zeros(0)
    if kept_vecs and all(v is not None for v in kept_vecs):
        vecs = np.stack(kept_vecs, axis=1)[:, order]
    else:
        vecs = np.zeros((0, 0))
    outcomes = [p[3] for p in parts]
    return SlicedResult(eigenvalues=vals, eigenvectors=vecs, converged=all(o.converged for o in outcomes),
                        spmv_total=sum(o.spmv_total for o in outcomes), slices=outcomes)
