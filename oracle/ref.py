"""ctypes binding of oracle/_ref/libadapoly_ref.so: the REFERENCE's own filter-path sources
(/root/reference/proj/src/cheb_filter.cpp + the headers it includes) compiled in place against the Eigen
stand-in (oracle/eigen_standin; Eigen is absent from this image) behind oracle/ref_capi.cpp.

Test infrastructure only: tests/test_ref_build.py checks the oracle restatement bit for bit against it.
The library is built by `make -C oracle` where /root/reference exists and travels prebuilt elsewhere;
`available()` says whether it is there.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libadapoly_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _ok(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: reference raised (code {rc})")


def _csr(a):
    return (np.ascontiguousarray(a.row_ptr, np.int64), np.ascontiguousarray(a.col_idx, np.int64),
            np.ascontiguousarray(a.values, np.float64))


def fill_gaussian(n, q, seed, stream):
    out = np.empty((n, q), order="F")
    _ok(lib().ref_fill_gaussian(C.c_int64(n), C.c_int64(q), C.c_uint64(seed), C.c_uint64(stream), _p(out)), "fill_gaussian")
    return out


def fill_rademacher(n, q, seed, stream):
    out = np.empty((n, q), order="F")
    _ok(lib().ref_fill_rademacher(C.c_int64(n), C.c_int64(q), C.c_uint64(seed), C.c_uint64(stream), _p(out)),
        "fill_rademacher")
    return out


def build_filter(a, b, bounds, k, m, damping="lanczos"):
    """Returns (coeffs, l1, l2, alpha, beta) of the reference's build_filter."""
    coeffs, params = np.empty(k + 1), np.empty(4)
    _ok(lib().ref_build_filter(C.c_double(a), C.c_double(b), C.c_double(bounds[0]), C.c_double(bounds[1]), C.c_int(k),
                               C.c_double(m), C.c_int(0 if damping == "lanczos" else 1), _p(coeffs), _p(params)),
        "build_filter")
    return coeffs, params[0], params[1], params[2], params[3]


def maspmm(a, t_i, t_k, b, c=None):
    b = np.asfortranarray(b, np.float64)
    out = np.zeros((a.n_rows, b.shape[1]), order="F") if c is None else np.array(c, np.float64, order="F", copy=True)
    rp, ci, v = _csr(a)
    _ok(lib().ref_maspmm(C.c_int64(a.n_rows), C.c_int64(a.n_cols), _p(rp), _p(ci), _p(v), C.c_int64(t_i),
                         C.c_int64(t_k), _p(b), C.c_int64(b.shape[1]), _p(out)), "maspmm")
    return out


def clenshaw_apply(coeffs, k_max, l1, l2, a, t_i, t_k, x, degree):
    """(Y, spmv_count) of the reference's clenshaw_apply on csr_to_tiled(A, t_i, t_k)."""
    x = np.asfortranarray(x, np.float64)
    y = np.empty(x.shape, order="F")
    rp, ci, v = _csr(a)
    c = np.ascontiguousarray(coeffs, np.float64)
    cnt = C.c_int64(0)
    _ok(lib().ref_clenshaw_apply(C.c_int64(a.n_rows), _p(rp), _p(ci), _p(v), C.c_int64(t_i), C.c_int64(t_k), _p(c),
                                 C.c_int(k_max), C.c_double(l1), C.c_double(l2), _p(x), C.c_int64(x.shape[1]),
                                 C.c_int(degree), _p(y), C.byref(cnt)), "clenshaw_apply")
    return y, cnt.value


def csr_spmv(a, x):
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(a.n_rows)
    rp, ci, v = _csr(a)
    _ok(lib().ref_csr_spmv(C.c_int64(a.n_rows), C.c_int64(a.n_cols), _p(rp), _p(ci), _p(v), _p(x), _p(y)), "csr_spmv")
    return y


def naive_spmm(a, b):
    b = np.asfortranarray(b, np.float64)
    c = np.empty((a.n_rows, b.shape[1]), order="F")
    rp, ci, v = _csr(a)
    _ok(lib().ref_naive_spmm(C.c_int64(a.n_rows), C.c_int64(a.n_cols), _p(rp), _p(ci), _p(v), _p(b),
                             C.c_int64(b.shape[1]), _p(c)), "naive_spmm")
    return c


def eval_filter(coeffs, k_max, l1, l2, x, degree):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    c = np.ascontiguousarray(coeffs, np.float64)
    clamped = C.c_int64(0)
    _ok(lib().ref_eval_filter(_p(c), C.c_int(k_max), C.c_double(l1), C.c_double(l2), _p(x), C.c_int64(len(x)),
                              C.c_int(degree), _p(out), C.byref(clamped)), "eval_filter_scalar")
    return out, clamped.value


def initial_degree(alpha, beta, c):
    out = C.c_int()
    _ok(lib().ref_initial_degree(C.c_double(alpha), C.c_double(beta), C.c_double(c), C.byref(out)), "initial_degree")
    return out.value


def adaptive_degree(coeffs, k_max, l1, l2, ritz, e_i, tau_a):
    r = np.ascontiguousarray(ritz, np.float64)
    c = np.ascontiguousarray(coeffs, np.float64)
    out = C.c_int()
    _ok(lib().ref_adaptive_degree(_p(c), C.c_int(k_max), C.c_double(l1), C.c_double(l2), _p(r), C.c_int64(len(r)),
                                  C.c_int64(e_i), C.c_double(tau_a), C.byref(out)), "adaptive_degree")
    return out.value


class Tiled:
    """The reference's TiledMatrix (csr_to_tiled, tiled_matrix.hpp:58-94) kept alive for timing."""

    def __init__(self, a, t_i=256, t_k=64):
        rp, ci, v = _csr(a)
        lib().ref_tiled_create.restype = C.c_void_p
        self.h = lib().ref_tiled_create(C.c_int64(a.n_rows), _p(rp), _p(ci), _p(v), C.c_int64(t_i), C.c_int64(t_k))
        if not self.h:
            raise RuntimeError("csr_to_tiled: reference raised")

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_tiled_destroy(C.c_void_p(self.h))
            self.h = None


def bench_clenshaw_steps(t: Tiled, q, steps):
    """(seconds, checksum) of `steps` middle Clenshaw steps: the reference's maspmm on its own tiling + the
    one-pass array update (ref_capi.cpp), on all OpenMP threads."""
    sec, cs = C.c_double(), C.c_double()
    _ok(lib().ref_bench_clenshaw_steps(C.c_void_p(t.h), C.c_int64(q), C.c_int(steps), C.byref(sec), C.byref(cs)),
        "bench_clenshaw_steps")
    return sec.value, cs.value
