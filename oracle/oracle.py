"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle (oracle.cpp).

The oracle restates the reference's hot path on the CPU (see the header of
oracle/oracle.cpp for what is restated and how it is pinned). Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU legs may import this module; the
product package ``paper_2604_00914_b200`` never does.

Dense operands cross this boundary column-major (Eigen's default storage,
``proj/include/adapoly/types.hpp:13-20``), i.e. numpy arrays in Fortran order.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

CONFIG, DIMENSION, NOT_PD, PARSE, RUNTIME = 1, 2, 3, 4, 5


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ConfigError(OracleError):
    pass


class DimensionError(OracleError):
    pass


_EXC = {CONFIG: ConfigError, DIMENSION: DimensionError}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


class Filter(C.Structure):
    _fields_ = [
        ("interval_a", C.c_double), ("interval_b", C.c_double),
        ("alpha", C.c_double), ("beta", C.c_double),
        ("k_max", C.c_int), ("m", C.c_double), ("l1", C.c_double), ("l2", C.c_double),
        ("lambda_min", C.c_double), ("lambda_max", C.c_double), ("active_degree", C.c_int),
    ]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P, I64, U64, D, I = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_set_threads": (None, [I]),
            "orc_max_threads": (I, []),
            "orc_philox_block": (None, [U64, U64, U64, P]),
            "orc_philox_raw": (None, [P, P, P]),
            "orc_fill_gaussian": (None, [P, I64, I64, U64, U64]),
            "orc_fill_rademacher": (None, [P, I64, I64, U64, U64]),
            "orc_gaussian": (D, [U64, U64, U64]),
            "orc_gaussian_range": (None, [U64, U64, U64, I64, P]),
            "orc_uniform_range": (None, [U64, U64, U64, I64, P]),
            "orc_mt_create": (P, [U64]),
            "orc_mt_destroy": (None, [P]),
            "orc_mt_next": (U64, [P]),
            "orc_mt_uniform": (D, [P, D, D]),
            "orc_mt_bernoulli": (I, [P, D]),
            "orc_mt_uniform_int": (I64, [P, I64, I64]),
            "orc_csr_from_triplets": (I, [I64, I64, I64, P, P, P, P]),
            "orc_random_csr": (P, [I64, I64, D, U64]),
            "orc_random_symmetric": (P, [I64, D, U64]),
            "orc_csr_wrap": (P, [I64, I64, P, P, P]),
            "orc_csr_destroy": (None, [P]),
            "orc_csr_dims": (None, [P, P, P, P]),
            "orc_csr_export": (None, [P, P, P, P]),
            "orc_zcsr_wrap": (P, [I64, I64, P, P, P]),
            "orc_zcsr_destroy": (None, [P]),
            "orc_tiled_create": (I, [P, I64, I64, P]),
            "orc_ztiled_create": (I, [P, I64, I64, P]),
            "orc_tiled_destroy": (None, [P]),
            "orc_ztiled_destroy": (None, [P]),
            "orc_tiled_sizes": (None, [P, P, P, P]),
            "orc_tiled_export": (None, [P, P, P, P, P, P]),
            "orc_maspmm": (I, [P, P, I64, P]),
            "orc_maspmm_shapes": (I, [P, I64, I64, I64, I64, I64, I64]),
            "orc_naive_spmm": (I, [P, P, I64, P]),
            "orc_csr_spmv": (I, [P, P, P]),
            "orc_step_coeffs": (I, [D, D, I, P]),
            "orc_lanczos_damping": (I, [I, D, P]),
            "orc_jackson_damping": (I, [I, P]),
            "orc_build_filter": (I, [D, D, D, D, I, D, I, P, P]),
            "orc_eval_filter_scalar": (D, [P, P, D, I]),
            "orc_eval_filter_vector": (I, [P, P, P, I64, I, P, P]),
            "orc_initial_degree": (I, [D, D, D, P]),
            "orc_adaptive_degree": (I, [P, P, P, I64, I64, D, P]),
            "orc_clenshaw_apply": (I, [P, I, D, D, P, P, I64, I64, I, P, P]),
            "orc_zclenshaw_apply": (I, [P, I, D, D, P, P, I64, I64, I, P, P]),
            "orc_estimate_eigcount": (I, [P, I, D, D, P, I64, U64, P, P]),
            "orc_bench_clenshaw_steps": (I, [P, I64, I, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        msg = lib().orc_last_error().decode()
        raise _EXC.get(status, OracleError)(status, msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def max_threads() -> int:
    return lib().orc_max_threads()


# ------------------------------------------------------------------ philox ---
def philox_block(seed: int, stream: int, counter: int) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    lib().orc_philox_block(seed, stream, counter, _ptr(out))
    return out


def philox_raw(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox_raw(_ptr(c), _ptr(k), _ptr(out))
    return out


def fill_gaussian(n: int, q: int, seed: int, stream: int) -> np.ndarray:
    out = np.empty((n, q), np.float64, order="F")
    lib().orc_fill_gaussian(_ptr(out), n, q, seed, stream)
    return out


def fill_rademacher(n: int, q: int, seed: int, stream: int) -> np.ndarray:
    out = np.empty((n, q), np.float64, order="F")
    lib().orc_fill_rademacher(_ptr(out), n, q, seed, stream)
    return out


def gaussian_range(seed: int, stream: int, first: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    lib().orc_gaussian_range(seed, stream, first, count, _ptr(out))
    return out


def uniform_range(seed: int, stream: int, first: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    lib().orc_uniform_range(seed, stream, first, count, _ptr(out))
    return out


class MT19937_64:
    """libstdc++ std::mt19937_64 with its distributions (test generators)."""

    def __init__(self, seed: int):
        self.h = lib().orc_mt_create(seed)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_mt_destroy(self.h)
            self.h = None

    def __call__(self) -> int:
        return lib().orc_mt_next(self.h)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return lib().orc_mt_uniform(self.h, lo, hi)

    def bernoulli(self, p: float = 0.5) -> bool:
        return bool(lib().orc_mt_bernoulli(self.h, p))

    def uniform_int(self, lo: int, hi: int) -> int:
        return lib().orc_mt_uniform_int(self.h, lo, hi)


# --------------------------------------------------------------------- CSR ---
@dataclass
class Csr:
    """Host CSR (int64 indices, sorted columns) -- CsrMatrix (csr_matrix.hpp:22-117)."""

    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray  # float64, or complex128 for Hermitian inputs

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def is_complex(self) -> bool:
        return np.iscomplexobj(self.values)

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols), self.values.dtype)
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        np.add.at(d, (rows, self.col_idx), self.values)
        return d

    @staticmethod
    def from_triplets(rows: int, cols: int, r, c, v) -> "Csr":
        r = np.ascontiguousarray(r, np.int64)
        c = np.ascontiguousarray(c, np.int64)
        v = np.ascontiguousarray(v, np.float64)
        h = C.c_void_p()
        _check(lib().orc_csr_from_triplets(rows, cols, len(v), _ptr(r), _ptr(c), _ptr(v), C.byref(h)))
        return _csr_take(h)


def _csr_take(h) -> Csr:
    L = lib()
    rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    L.orc_csr_dims(h, C.byref(rows), C.byref(cols), C.byref(nnz))
    rp = np.empty(rows.value + 1, np.int64)
    ci = np.empty(nnz.value, np.int64)
    v = np.empty(nnz.value, np.float64)
    L.orc_csr_export(h, _ptr(rp), _ptr(ci), _ptr(v))
    L.orc_csr_destroy(h)
    return Csr(rows.value, cols.value, rp, ci, v)


def random_csr(rows: int, cols: int, density: float, seed: int) -> Csr:
    """test_support::random_csr (proj/tests/support/test_matrices.hpp:38-48), bit for bit."""
    return _csr_take(lib().orc_random_csr(rows, cols, density, seed))


def random_symmetric(n: int, density: float, seed: int) -> Csr:
    """test_support::random_symmetric (test_matrices.hpp:51-65), bit for bit."""
    return _csr_take(lib().orc_random_symmetric(n, density, seed))


def make_diag(d) -> Csr:
    d = np.asarray(d, np.float64)
    n = len(d)
    return Csr(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), d.copy())


class _Handle:
    def __init__(self, a: Csr):
        self.a = a
        self._rp = np.ascontiguousarray(a.row_ptr, np.int64)
        self._ci = np.ascontiguousarray(a.col_idx, np.int64)
        if a.is_complex:
            self._v = np.ascontiguousarray(a.values, np.complex128).view(np.float64)
            self.h = lib().orc_zcsr_wrap(a.n_rows, a.n_cols, _ptr(self._rp), _ptr(self._ci), _ptr(self._v))
        else:
            self._v = np.ascontiguousarray(a.values, np.float64)
            self.h = lib().orc_csr_wrap(a.n_rows, a.n_cols, _ptr(self._rp), _ptr(self._ci), _ptr(self._v))

    def __del__(self):
        if getattr(self, "h", None):
            (lib().orc_zcsr_destroy if self.a.is_complex else lib().orc_csr_destroy)(self.h)
            self.h = None


class Tiled:
    """TiledMatrix built by csr_to_tiled (tiled_matrix.hpp:58-94)."""

    def __init__(self, a: Csr, t_i: int = 256, t_k: int = 64):
        self.csr = _Handle(a)
        self.n_rows, self.n_cols, self.t_i, self.t_k = a.n_rows, a.n_cols, t_i, t_k
        self.is_complex = a.is_complex
        h = C.c_void_p()
        fn = lib().orc_ztiled_create if a.is_complex else lib().orc_tiled_create
        _check(fn(self.csr.h, t_i, t_k, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            (lib().orc_ztiled_destroy if self.is_complex else lib().orc_tiled_destroy)(self.h)
            self.h = None

    def export(self):
        ns, nb, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        lib().orc_tiled_sizes(self.h, C.byref(ns), C.byref(nb), C.byref(nnz))
        act = np.empty(nb.value + 1, np.int64)
        csp = np.empty(ns.value + 1, np.int64)
        ci = np.empty(ns.value, np.int64)
        ri = np.empty(nnz.value, np.int64)
        v = np.empty(nnz.value, np.float64)
        lib().orc_tiled_export(self.h, _ptr(act), _ptr(csp), _ptr(ci), _ptr(ri), _ptr(v))
        return dict(act_colseg=act, colseg_ptr=csp, col_idx=ci, row_idx=ri, values=v)


def maspmm(t: Tiled, b: np.ndarray, c: np.ndarray | None = None) -> np.ndarray:
    """C += A B through the block layout; returns C (column-major)."""
    b = np.asfortranarray(b, np.float64)
    k = b.shape[1]
    if b.shape[0] != t.n_cols:
        raise DimensionError(DIMENSION, "maspmm: shape mismatch")
    c = np.zeros((t.n_rows, k), order="F") if c is None else np.array(c, np.float64, order="F", copy=True)
    _check(lib().orc_maspmm(t.h, _ptr(b), k, _ptr(c)))
    return c


def maspmm_shapes(t: Tiled, b_shape, c_shape) -> None:
    _check(lib().orc_maspmm_shapes(t.h, *b_shape, *c_shape))


def naive_spmm(a: Csr, b: np.ndarray) -> np.ndarray:
    h = _Handle(a)
    b = np.asfortranarray(b, np.float64)
    c = np.empty((a.n_rows, b.shape[1]), order="F")
    _check(lib().orc_naive_spmm(h.h, _ptr(b), b.shape[1], _ptr(c)))
    return c


def csr_spmv(a: Csr, x: np.ndarray) -> np.ndarray:
    h = _Handle(a)
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(a.n_rows)
    _check(lib().orc_csr_spmv(h.h, _ptr(x), _ptr(y)))
    return y


# ------------------------------------------------------------------- filter ---
def chebyshev_step_coeffs(alpha: float, beta: float, k: int) -> np.ndarray:
    out = np.empty(max(k, 0) + 1)
    _check(lib().orc_step_coeffs(alpha, beta, k, _ptr(out)))
    return out


def lanczos_damping(k: int, m: float) -> np.ndarray:
    out = np.empty(max(k, 0) + 1)
    _check(lib().orc_lanczos_damping(k, m, _ptr(out)))
    return out


def jackson_damping(k: int) -> np.ndarray:
    out = np.empty(max(k, 0) + 1)
    _check(lib().orc_jackson_damping(k, _ptr(out)))
    return out


@dataclass
class ChebFilter:
    """ChebFilter (proj/include/adapoly/cheb_filter.hpp:41-66)."""

    interval_a: float
    interval_b: float
    alpha: float
    beta: float
    k_max: int
    m: float
    l1: float
    l2: float
    lambda_min: float
    lambda_max: float
    coeffs: np.ndarray = field(repr=False)
    active_degree: int = 0

    def map(self, x):
        return self.l1 * x + self.l2

    def _struct(self) -> Filter:
        return Filter(self.interval_a, self.interval_b, self.alpha, self.beta, self.k_max, self.m,
                      self.l1, self.l2, self.lambda_min, self.lambda_max, self.active_degree)


def build_filter(a: float, b: float, bounds, k: int, m: float, damping: str = "lanczos") -> ChebFilter:
    f = Filter()
    coeffs = np.empty(max(k, 0) + 1)
    _check(lib().orc_build_filter(a, b, bounds[0], bounds[1], k, m, 0 if damping == "lanczos" else 1,
                                  C.byref(f), _ptr(coeffs)))
    return ChebFilter(f.interval_a, f.interval_b, f.alpha, f.beta, f.k_max, f.m, f.l1, f.l2,
                      f.lambda_min, f.lambda_max, coeffs, f.active_degree)


def eval_filter_scalar(f: ChebFilter, x, degree: int):
    s = f._struct()
    c = np.ascontiguousarray(f.coeffs, np.float64)
    if np.isscalar(x):
        return lib().orc_eval_filter_scalar(C.byref(s), _ptr(c), float(x), degree)
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    clamped = C.c_int64(0)
    _check(lib().orc_eval_filter_vector(C.byref(s), _ptr(c), _ptr(x), len(x), degree, _ptr(out), C.byref(clamped)))
    return out, clamped.value


def initial_degree(alpha: float, beta: float, c: float) -> int:
    out = C.c_int()
    _check(lib().orc_initial_degree(alpha, beta, c, C.byref(out)))
    return out.value


def adaptive_degree(f: ChebFilter, ritz, e_i: int, tau_a: float) -> int:
    s = f._struct()
    c = np.ascontiguousarray(f.coeffs, np.float64)
    r = np.ascontiguousarray(ritz, np.float64)
    out = C.c_int()
    _check(lib().orc_adaptive_degree(C.byref(s), _ptr(c), _ptr(r), len(r), e_i, tau_a, C.byref(out)))
    return out.value


def clenshaw_apply(f: ChebFilter, t: Tiled, x: np.ndarray, degree: int, spmv: list | None = None) -> np.ndarray:
    """rho(l(A)) X, column-major in/out (cheb_filter.cpp:129-179), bitwise restatement."""
    c = np.ascontiguousarray(f.coeffs, np.float64)
    cnt = C.c_int64(spmv[0] if spmv else 0)
    if t.is_complex:
        x = np.asfortranarray(x, np.complex128)
        out = np.zeros(x.shape, np.complex128, order="F")
        fn = lib().orc_zclenshaw_apply
    else:
        x = np.asfortranarray(x, np.float64)
        out = np.zeros(x.shape, np.float64, order="F")
        fn = lib().orc_clenshaw_apply
    _check(fn(_ptr(c), f.k_max, f.l1, f.l2, t.h, _ptr(x), x.shape[0], x.shape[1], degree, _ptr(out),
              C.byref(cnt)))
    if spmv is not None:
        spmv[0] = cnt.value
    return out


def estimate_eigcount(t: Tiled, f: ChebFilter, probes: int, seed: int, spmv: list | None = None) -> float:
    c = np.ascontiguousarray(f.coeffs, np.float64)
    out = C.c_double()
    cnt = C.c_int64(spmv[0] if spmv else 0)
    _check(lib().orc_estimate_eigcount(_ptr(c), f.k_max, f.l1, f.l2, t.h, probes, seed, C.byref(out), C.byref(cnt)))
    if spmv is not None:
        spmv[0] = cnt.value
    return out.value


def bench_clenshaw_steps(t: Tiled, q: int, steps: int):
    """Seconds for `steps` middle Clenshaw steps (maspmm + update) on block-layout operands."""
    sec, cs = C.c_double(), C.c_double()
    _check(lib().orc_bench_clenshaw_steps(t.h, q, steps, C.byref(sec), C.byref(cs)))
    return sec.value, cs.value


def forward_filter_apply(f: ChebFilter, a_dense: np.ndarray, x: np.ndarray, degree: int) -> np.ndarray:
    """Forward-accumulation oracle (proj/tests/test_cheb_filter.cpp:21-38), dense numpy."""
    n = a_dense.shape[0]
    t = f.l1 * a_dense + f.l2 * np.eye(n)
    acc = f.coeffs[0] * x
    if degree >= 1:
        t_prev = x
        t_cur = t @ x
        acc = acc + f.coeffs[1] * t_cur
        for j in range(2, degree + 1):
            t_next = 2.0 * (t @ t_cur) - t_prev
            acc = acc + f.coeffs[j] * t_next
            t_prev, t_cur = t_cur, t_next
    return acc
