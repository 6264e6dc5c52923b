"""Chebyshev step-function filter construction (host side of the hot path).

Mirrors proj/include/adapoly/cheb_filter.hpp / proj/src/cheb_filter.cpp: the
functions keep the reference's names, argument meaning and error behaviour
(ConfigError on invalid input). The arithmetic runs in libadp_b200.so
(csrc/filter_host.cpp) so the coefficient bits match the reference's.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._native import FilterInfo, check, lib


@dataclass
class SpectrumBounds:
    """SpectrumBounds (cheb_filter.hpp:13-22)."""

    lambda_min: float = 0.0
    lambda_max: float = 0.0

    def scale(self) -> float:
        return max(abs(self.lambda_min), abs(self.lambda_max))


@dataclass
class ChebFilter:
    """ChebFilter (cheb_filter.hpp:41-66): damped step-function expansion."""

    interval_a: float
    interval_b: float
    alpha: float
    beta: float
    k_max: int
    m: float
    l1: float
    l2: float
    bounds: SpectrumBounds
    coeffs: np.ndarray = field(repr=False)
    active_degree: int = 0

    def map(self, x):
        return self.l1 * x + self.l2

    def map_clamped(self, x: float) -> float:
        t = self.map(x)
        return -1.0 if t < -1.0 else (1.0 if t > 1.0 else t)

    def info(self) -> FilterInfo:
        return FilterInfo(self.interval_a, self.interval_b, self.alpha, self.beta, self.k_max, self.m, self.l1,
                          self.l2, self.bounds.lambda_min, self.bounds.lambda_max, self.active_degree)

    def coeff_array(self) -> np.ndarray:
        return np.ascontiguousarray(self.coeffs, np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def chebyshev_step_coeffs(alpha: float, beta: float, k: int) -> np.ndarray:
    """chebyshev_step_coeffs (cheb_filter.cpp:21-37)."""
    out = np.empty(max(int(k), 0) + 1)
    check(lib().adp_step_coeffs(alpha, beta, int(k), _ptr(out)))
    return out


def lanczos_damping(k: int, m: float) -> np.ndarray:
    """lanczos_damping (cheb_filter.cpp:39-49)."""
    out = np.empty(max(int(k), 0) + 1)
    check(lib().adp_lanczos_damping(int(k), m, _ptr(out)))
    return out


def jackson_damping(k: int) -> np.ndarray:
    """jackson_damping (cheb_filter.cpp:51-61)."""
    out = np.empty(max(int(k), 0) + 1)
    check(lib().adp_jackson_damping(int(k), _ptr(out)))
    return out


def build_filter(a: float, b: float, bounds, k: int, m: float, damping: str = "lanczos") -> ChebFilter:
    """build_filter (cheb_filter.cpp:63-94); bounds is a SpectrumBounds or (lmin, lmax)."""
    if not isinstance(bounds, SpectrumBounds):
        bounds = SpectrumBounds(float(bounds[0]), float(bounds[1]))
    info = FilterInfo()
    coeffs = np.empty(max(int(k), 0) + 1)
    kind = {"lanczos": 0, "jackson": 1}[damping]
    check(lib().adp_build_filter(a, b, bounds.lambda_min, bounds.lambda_max, int(k), m, kind, C.byref(info),
                                 _ptr(coeffs)))
    return ChebFilter(info.interval_a, info.interval_b, info.alpha, info.beta, info.k_max, info.m, info.l1, info.l2,
                      SpectrumBounds(info.lambda_min, info.lambda_max), coeffs, info.active_degree)


def eval_filter_scalar(f: ChebFilter, x, degree: int, clamped: list | None = None):
    """eval_filter_scalar (cheb_filter.cpp:96-127): scalar in -> float out; array in -> array out.

    ``clamped`` (a one-element list) accumulates the number of clamped arguments.
    """
    scalar = np.isscalar(x)
    xs = np.ascontiguousarray(np.atleast_1d(x), np.float64)
    out = np.empty_like(xs)
    cnt = C.c_int64(clamped[0] if clamped else 0)
    info = f.info()
    coeffs = f.coeff_array()
    # The scalar overload (cheb_filter.cpp:96) has no range check; the vector one does.
    deg = int(degree)
    if scalar and not (0 <= deg <= f.k_max):
        deg = min(max(deg, 0), f.k_max)
    check(lib().adp_eval_filter(C.byref(info), _ptr(coeffs), _ptr(xs), len(xs), deg, _ptr(out), C.byref(cnt)))
    if clamped is not None:
        clamped[0] = cnt.value
    return float(out[0]) if scalar else out


def initial_degree(alpha: float, beta: float, c: float) -> int:
    """initial_degree (cheb_filter.cpp:181-187): max(ceil(C / (alpha - beta)) - 1, 1)."""
    out = C.c_int32()
    check(lib().adp_initial_degree(alpha, beta, c, C.byref(out)))
    return out.value


def adaptive_degree(f: ChebFilter, ritz, e_i: int, tau_a: float) -> int:
    """adaptive_degree (cheb_filter.cpp:189-219)."""
    r = np.ascontiguousarray(ritz, np.float64)
    out = C.c_int32()
    info = f.info()
    coeffs = f.coeff_array()
    check(lib().adp_adaptive_degree(C.byref(info), _ptr(coeffs), _ptr(r), len(r), int(e_i), tau_a, C.byref(out)))
    return out.value
