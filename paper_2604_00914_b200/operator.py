"""Device operator API: context, device CSR, clenshaw_apply and maspmm.

These are the reference's operator-level entry points
(proj/include/adapoly/cheb_filter.hpp:84-86 ``clenshaw_apply``,
proj/include/adapoly/tiled_matrix.hpp:184-186 ``maspmm``) over the C-ABI of
libadp_b200.so. Host numpy operands are column-major like the reference's
Eigen matrices; device operands are torch CUDA tensors, row-major n x q.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import ADP_C128, ADP_COL_MAJOR, ADP_F64, ADP_ROW_MAJOR, ConfigError, DimensionError, check, lib
from .filter import ChebFilter
from .sparse import CsrMatrix


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Context:
    """adp_ctx: one CUDA device, a stream, library handles and workspace."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().adp_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = int(device)

    def close(self):
        if getattr(self, "h", None):
            check(lib().adp_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream) -> None:
        """Queue work on an existing cudaStream_t (int handle or torch.cuda.Stream; 0 = legacy default
        stream, torch's default). None = the context's own non-blocking stream."""
        if stream is None:
            handle = lib().adp_ctx_own_stream(self.h) or 0
        else:
            handle = int(getattr(stream, "cuda_stream", stream))
        check(lib().adp_ctx_set_stream(self.h, C.c_void_p(handle)))

    def synchronize(self) -> None:
        check(lib().adp_ctx_synchronize(self.h))

    @property
    def launch_count(self) -> int:
        return int(lib().adp_ctx_launch_count(self.h))

    def set_panel(self, cols: int) -> None:
        check(lib().adp_ctx_set_panel(self.h, int(cols)))

    def set_tuning(self, variant: int) -> None:
        """Kernel family: 0 automatic, 1 row, 2 lean, 3 line, 4 cube, 5 plane sweep (adp.h)."""
        check(lib().adp_ctx_set_tuning(self.h, int(variant)))

    @property
    def last_step_kernel(self) -> int:
        """Family of the last fused-step launch (1 row, 2 lean, 3 line, 4 cube, 5 plane sweep)."""
        return int(lib().adp_ctx_last_step_kernel(self.h))


_default_ctx: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


class DeviceCsr:
    """adp_csr: a CSR operator resident in HBM (int32 columns, fp64 / complex128 values).

    Replaces the reference's TiledMatrix (tiled_matrix.hpp:23-52): the row-block /
    column-segment regrouping was a CPU-cache device; the GPU kernel walks CSR rows
    directly in the same ascending-column accumulation order.
    """

    def __init__(self, a: CsrMatrix, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.n_rows, self.n_cols = int(a.n_rows), int(a.n_cols)
        self.is_complex = a.is_complex
        rp = np.ascontiguousarray(a.row_ptr, np.int64)
        ci = np.ascontiguousarray(a.col_idx, np.int64)
        if self.is_complex:
            v = np.ascontiguousarray(a.values, np.complex128)
            dt = ADP_C128
        else:
            v = np.ascontiguousarray(a.values, np.float64)
            dt = ADP_F64
        h = C.c_void_p()
        check(lib().adp_csr_create(self.ctx.h, self.n_rows, self.n_cols, _ptr(rp), _ptr(ci), _ptr(v), dt,
                                   C.byref(h)))
        self.h = h
        self.nnz = int(rp[-1])

    @classmethod
    def from_device(cls, n_rows: int, n_cols: int, row_ptr, col_idx, values, ctx: Context | None = None) -> "DeviceCsr":
        """adp_csr_create_device: an operator from CUDA tensors (int64 row_ptr, int32 col_idx, float64 or
        complex128 values) already on ctx's device -- for operators generated on the GPU (config 5).
        Validated on the device like CsrMatrix::validate; the tensors are copied."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        if str(values.dtype) not in ("torch.float64", "torch.complex128"):
            raise ConfigError("DeviceCsr.from_device: values must be float64 or complex128")
        if str(row_ptr.dtype) != "torch.int64" or str(col_idx.dtype) != "torch.int32":
            raise ConfigError("DeviceCsr.from_device: row_ptr must be int64 and col_idx int32")
        for t in (row_ptr, col_idx, values):
            if not t.is_cuda or not t.is_contiguous():
                raise ConfigError("DeviceCsr.from_device: arrays must be contiguous CUDA tensors")
        if row_ptr.numel() != self.n_rows + 1 or col_idx.numel() != values.numel():
            raise DimensionError("DeviceCsr.from_device: array sizes do not match the dimensions")
        self.is_complex = str(values.dtype) == "torch.complex128"
        self.nnz = int(col_idx.numel())
        h = C.c_void_p()
        check(lib().adp_csr_create_device(self.ctx.h, self.n_rows, self.n_cols, self.nnz, C.c_void_p(row_ptr.data_ptr()),
                                          C.c_void_p(col_idx.data_ptr()), C.c_void_p(values.data_ptr()),
                                          ADP_C128 if self.is_complex else ADP_F64, C.byref(h)))
        self.h = h
        return self

    @property
    def dtype(self):
        return np.complex128 if self.is_complex else np.float64

    def stencil(self) -> tuple[int, tuple[int, int, int]]:
        """(kind, (nx, ny, nz)) if the operator is a constant-coefficient radius-1 stencil (27 box /
        7 star; the plane-sweep kernel's precondition, verified against the CSR), else (0, (0, 0, 0))."""
        kind = C.c_int32()
        dims = (C.c_int64 * 3)()
        check(lib().adp_csr_stencil(self.h, C.byref(kind), dims))
        return int(kind.value), (int(dims[0]), int(dims[1]), int(dims[2]))

    def close(self):
        if getattr(self, "h", None):
            check(lib().adp_csr_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def clenshaw_apply(f: ChebFilter, a: DeviceCsr, x: np.ndarray, degree: int, spmv_count: list | None = None,
                   layout: str = "col") -> np.ndarray:
    """rho(l(A)) X on the GPU with host operands (cheb_filter.cpp:129-179).

    Same contract as the reference: ConfigError for a degree outside [0, k_max],
    DimensionError when X's row count differs from A's, trailing zero
    coefficients reduce the degree, ``spmv_count[0] += effective_degree * q``.
    Column-major (Fortran) output, bitwise equal to the reference arithmetic.
    """
    if x.ndim != 2:
        raise DimensionError("clenshaw_apply: X must be a matrix")
    dt = a.dtype
    n, q = x.shape
    if layout == "col":
        xs = np.asfortranarray(x, dt)
        out = np.empty((a.n_rows if n == a.n_cols else n, q), dt, order="F")
        ldx, ldy, lay = max(n, 1), max(out.shape[0], 1), ADP_COL_MAJOR
    else:
        xs = np.ascontiguousarray(x, dt)
        out = np.empty((n, q), dt)
        ldx, ldy, lay = max(q, 1), max(q, 1), ADP_ROW_MAJOR
    coeffs = f.coeff_array()
    cnt = C.c_int64(spmv_count[0] if spmv_count else 0)
    check(lib().adp_filter_apply(a.ctx.h, a.h, _ptr(coeffs), f.k_max, f.l1, f.l2, int(degree), _ptr(xs), n, ldx, q,
                                 lay, _ptr(out), ldy, C.byref(cnt)))
    if spmv_count is not None:
        spmv_count[0] = cnt.value
    return out


def clenshaw_apply_device(f: ChebFilter, a: DeviceCsr, x, degree: int, out=None, spmv_count: list | None = None):
    """Device-resident variant: x, out are torch CUDA tensors (n x q, row-major, stride(1) == 1).

    Work is queued on torch's current stream (no host synchronisation).
    """
    import torch

    if out is None:
        out = torch.empty_like(x)
    if x.dim() != 2 or x.stride(1) != 1 or out.stride(1) != 1:
        raise DimensionError("clenshaw_apply_device: operands must be row-major matrices")
    a.ctx.set_stream(torch.cuda.current_stream(x.device))
    coeffs = f.coeff_array()
    cnt = C.c_int64(spmv_count[0] if spmv_count else 0)
    n, q = x.shape
    check(lib().adp_filter_apply_device(a.ctx.h, a.h, _ptr(coeffs), f.k_max, f.l1, f.l2, int(degree),
                                        C.c_void_p(x.data_ptr()), n, x.stride(0), q, C.c_void_p(out.data_ptr()),
                                        out.stride(0), C.byref(cnt)))
    if spmv_count is not None:
        spmv_count[0] = cnt.value
    return out


def maspmm(a: DeviceCsr, b: np.ndarray, c: np.ndarray | None = None, accumulate: bool = True) -> np.ndarray:
    """C += A B (tiled_matrix.hpp:184-210) with host column-major operands; returns C.

    With c=None a zero C is used (the reference's set_zero() + maspmm).
    """
    dt = a.dtype
    b = np.asfortranarray(b, dt)
    k = b.shape[1]
    if c is None:
        c = np.zeros((a.n_rows, k), dt, order="F")
        acc = 0
    else:
        if c.shape != (a.n_rows, k):
            raise DimensionError("maspmm: shape mismatch")
        c = np.array(c, dt, order="F", copy=True)
        acc = 1 if accumulate else 0
    check(lib().adp_spmm(a.ctx.h, a.h, _ptr(b), b.shape[0], max(b.shape[0], 1), k, ADP_COL_MAJOR, _ptr(c),
                         max(a.n_rows, 1), acc))
    return c


def csr_spmv_device(a: DeviceCsr, x, y):
    """y = A x (csr_matrix.hpp:122-134: sequential CSR-order accumulation) on torch CUDA fp64 vectors."""
    import torch

    if a.is_complex:
        raise ConfigError("csr_spmv: real operators only")
    if x.numel() != a.n_cols or y.numel() != a.n_rows or not (x.is_contiguous() and y.is_contiguous()):
        raise DimensionError("csr_spmv: vector sizes do not match the operator")
    a.ctx.set_stream(torch.cuda.current_stream(x.device))
    check(lib().adp_spmv_device(a.ctx.h, a.h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr())))
    return y


def maspmm_device(a: DeviceCsr, b, c, accumulate: bool = False):
    """C (+)= A B on torch CUDA tensors (row-major), queued on the current stream."""
    import torch

    a.ctx.set_stream(torch.cuda.current_stream(b.device))
    check(lib().adp_spmm_device(a.ctx.h, a.h, C.c_void_p(b.data_ptr()), b.shape[0], b.stride(0), b.shape[1],
                                C.c_void_p(c.data_ptr()), c.stride(0), 1 if accumulate else 0))
    return c
