"""Filter truncation-error bounds and the inspect-filter sweep.

Mirrors proj/include/adapoly/filter_bounds.hpp:8-30 (j_theta, c_m_constant,
undamped_bound, damped_bound, projector_bound -- computed by the C-ABI,
csrc/bounds.cpp) and the `inspect-filter` flow of proj/src/cli.cpp:198-235
(x, rho, |step - rho|, damped bound on a uniform sweep). Errors follow the
reference: ConfigError for out-of-range degrees, m <= 0 in C_m, empty angle
lists.
"""
from __future__ import annotations

import ctypes as C
import io
import math

import numpy as np

from ._native import ConfigError, check, lib
from .filter import ChebFilter, SpectrumBounds, build_filter, eval_filter_scalar


def _out(fn, *args) -> float:
    v = C.c_double(0.0)
    check(fn(*args, C.byref(v)))
    return v.value


def j_theta(theta: float, alpha: float, beta: float) -> float:
    """J(theta): reciprocal-sine sum; +inf where a denominator sine vanishes."""
    return _out(lib().adp_j_theta, float(theta), float(alpha), float(beta))


def c_m_constant(m: float) -> float:
    """C_m = int_0^pi (sin u)^(m-1) (sin u - u cos u) / u^(m+2) du (cached per m)."""
    return _out(lib().adp_c_m_constant, float(m))


def undamped_bound(theta: float, k: int, alpha: float, beta: float) -> float:
    return _out(lib().adp_undamped_bound, float(theta), int(k), float(alpha), float(beta))


def damped_bound(theta: float, k_i: int, k: int, m: float, alpha: float, beta: float) -> float:
    return _out(lib().adp_damped_bound, float(theta), int(k_i), int(k), float(m), float(alpha), float(beta))


def projector_bound(f: ChebFilter, eigen_thetas, k_i: int) -> float:
    """Bound on ||P - P_i||_2 from the angles arccos(l(lambda_j)) of the eigenvalues."""
    th = np.ascontiguousarray(np.atleast_1d(np.asarray(eigen_thetas, np.float64)))
    info = f.info()
    return _out(lib().adp_projector_bound, C.byref(info), th.ctypes.data_as(C.c_void_p), len(th), int(k_i))


def inspect_filter(a: float, b: float, bounds=(-1.0, 1.0), k: int = 100, m: float = 0.5,
                   degree: int | None = None, samples: int = 200, sweep=None) -> list[tuple[float, float, float, float]]:
    """The inspect-filter sweep (cli.cpp:198-235): rows (x, rho(x), |step(x) - rho(x)|, damped bound)."""
    lo, hi = float(bounds[0]), float(bounds[1])
    if not lo < hi:
        raise ConfigError("bounds must satisfy lo < hi")
    f = build_filter(a, b, SpectrumBounds(lo, hi), k, m)
    deg = k if degree is None else int(degree)
    if deg < 1 or deg > k:
        raise ConfigError("degree must lie in [1, k]")
    s_lo, s_hi = (lo, hi) if sweep is None else (float(sweep[0]), float(sweep[1]))
    if samples < 0:
        raise ConfigError("samples must be >= 0")
    rows = []
    for i in range(int(samples)):
        x = s_lo if samples == 1 else s_lo + (s_hi - s_lo) * float(i) / float(samples - 1)
        rho = eval_filter_scalar(f, x, deg)
        step = 1.0 if a < x < b else (0.5 if x == a or x == b else 0.0)
        theta = math.acos(f.map_clamped(x))
        rows.append((x, rho, abs(step - rho), damped_bound(theta, deg, k, m, f.alpha, f.beta)))
    return rows


def inspect_filter_csv(*args, **kwargs) -> str:
    """inspect_filter as the CLI's CSV text (header x,rho,error,bound; 17 significant digits)."""
    buf = io.StringIO()
    buf.write("x,rho,error,bound\n")
    for row in inspect_filter(*args, **kwargs):
        buf.write(",".join(_g17(v) for v in row) + "\n")
    return buf.getvalue()


def _g17(v: float) -> str:
    # std::ostream << setprecision(17): %.17g ('inf' / 'nan' as the C++ stream prints them)
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    if math.isnan(v):
        return "nan"
    return "%.17g" % v
