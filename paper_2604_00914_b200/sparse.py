"""Host CSR container, Matrix Market ingestion and seeded draws.

``CsrMatrix`` mirrors the reference's CsrMatrix (proj/include/adapoly/
csr_matrix.hpp:22-117): int64 row offsets / column indices, rows sorted by
column, duplicates summed, both triangles stored for symmetric operators.
Values are float64, or complex128 for Hermitian operators (an extension: the
reference is real-only).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._native import DimensionError, ParseError, check, lib


@dataclass
class CsrMatrix:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # int64[n_rows + 1]
    col_idx: np.ndarray  # int64[nnz]
    values: np.ndarray   # float64[nnz] or complex128[nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def is_complex(self) -> bool:
        return np.iscomplexobj(self.values)

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    @staticmethod
    def from_triplets(rows: int, cols: int, r, c, v) -> "CsrMatrix":
        """CsrMatrix::from_triplets (csr_matrix.hpp:34-62): sort by (row, col), sum duplicates."""
        r = np.asarray(r, np.int64)
        c = np.asarray(c, np.int64)
        v = np.asarray(v)
        if rows < 0 or cols < 0:
            raise DimensionError("negative matrix size")
        if len(r) and (r.min() < 0 or r.max() >= rows or c.min() < 0 or c.max() >= cols):
            raise DimensionError("triplet index out of bounds")
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        if len(r):
            new = np.ones(len(r), bool)
            new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
            starts = np.flatnonzero(new)
            v = np.add.reduceat(v, starts) if len(starts) != len(v) else v
            r, c = r[starts], c[starts]
        row_ptr = np.zeros(rows + 1, np.int64)
        np.add.at(row_ptr, r + 1, 1)
        row_ptr = np.cumsum(row_ptr)
        return CsrMatrix(rows, cols, row_ptr, c, np.ascontiguousarray(v))

    def validate(self) -> None:
        """CsrMatrix::validate (csr_matrix.hpp:101-116)."""
        rp, ci = self.row_ptr, self.col_idx
        if len(rp) != self.n_rows + 1:
            raise DimensionError("row_ptr length mismatch")
        if rp[0] != 0 or rp[-1] != len(self.values):
            raise DimensionError("row_ptr endpoints mismatch")
        if np.any(np.diff(rp) < 0):
            raise DimensionError("row_ptr not non-decreasing")
        if len(ci) and (ci.min() < 0 or ci.max() >= self.n_cols):
            raise DimensionError("column index out of range")
        if len(ci) > 1:
            same_row = np.repeat(np.arange(self.n_rows), np.diff(rp))
            bad = (same_row[1:] == same_row[:-1]) & (ci[1:] <= ci[:-1])
            if bad.any():
                raise DimensionError("columns not strictly increasing within a row")

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols), self.values.dtype)
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        np.add.at(d, (rows, self.col_idx), self.values)
        return d

    def is_symmetric(self) -> bool:
        """Exact (Hermitian, for complex) symmetry of the stored matrix (csr_matrix.hpp:82-98)."""
        if self.n_rows != self.n_cols:
            return False
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        fwd = np.lexsort((self.col_idx, rows))
        rev = np.lexsort((rows, self.col_idx))
        if not (np.array_equal(rows[fwd], self.col_idx[rev]) and np.array_equal(self.col_idx[fwd], rows[rev])):
            return False
        return bool(np.array_equal(self.values[fwd], np.conj(self.values[rev])))

    def spmv(self, x: np.ndarray) -> np.ndarray:
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        out = np.zeros(self.n_rows, np.result_type(self.values, x))
        np.add.at(out, rows, self.values * x[self.col_idx])
        return out


def parse_matrix_market(text: str) -> CsrMatrix:
    """parse_matrix_market (proj/src/matrix_market.cpp:22-89).

    Coordinate real / integer, general / symmetric, as in the reference, plus
    complex general / hermitian (the Hermitian extension). Symmetric and
    Hermitian storage is expanded to both triangles; errors are ParseError with
    the 1-based line number.
    """
    lines = text.splitlines()
    if not lines:
        raise ParseError("line 1: empty stream")
    banner = lines[0].split()
    while len(banner) < 5:
        banner.append("")
    tag, obj, fmt, fld, sym = (t.lower() for t in banner[:5])
    if tag != "%%matrixmarket":
        raise ParseError("line 1: missing %%MatrixMarket banner")
    if obj != "matrix":
        raise ParseError(f"line 1: unsupported object '{banner[1]}'")
    if fmt != "coordinate":
        raise ParseError(f"line 1: unsupported format '{banner[2]}' (coordinate required)")
    if fld not in ("real", "integer", "complex"):
        raise ParseError(f"line 1: unsupported field '{fld}' (real, integer or complex required)")
    if sym not in ("general", "symmetric", "hermitian"):
        raise ParseError(f"line 1: unsupported symmetry '{sym}'")
    cplx = fld == "complex"
    if sym == "hermitian" and not cplx:
        raise ParseError("line 1: hermitian symmetry requires the complex field")
    i = 1
    rows = cols = nnz = -1
    while i < len(lines):
        ln = lines[i]
        i += 1
        if not ln or ln[0] == "%":
            continue
        parts = ln.split()
        try:
            rows, cols, nnz = int(parts[0]), int(parts[1]), int(parts[2])
        except (ValueError, IndexError):
            raise ParseError(f"line {i}: malformed size line") from None
        if rows < 0 or cols < 0 or nnz < 0:
            raise ParseError(f"line {i}: malformed size line")
        break
    if rows < 0:
        raise ParseError(f"line {i + 1}: missing size line")
    r_l, c_l, v_l = [], [], []
    seen = 0
    while seen < nnz:
        if i >= len(lines):
            raise ParseError(f"line {i + 1}: unexpected end of stream, expected {nnz} entries, got {seen}")
        ln = lines[i]
        i += 1
        if not ln or ln[0] == "%":
            continue
        parts = ln.split()
        try:
            a, b = int(parts[0]), int(parts[1])
            v = complex(float(parts[2]), float(parts[3])) if cplx else float(parts[2])
        except (ValueError, IndexError):
            raise ParseError(f"line {i}: malformed entry") from None
        if a < 1 or a > rows or b < 1 or b > cols:
            raise ParseError(f"line {i}: index out of declared bounds")
        r_l.append(a - 1)
        c_l.append(b - 1)
        v_l.append(v)
        if sym != "general" and a != b:
            r_l.append(b - 1)
            c_l.append(a - 1)
            v_l.append(np.conj(v) if sym == "hermitian" else v)
        seen += 1
    while i < len(lines):
        ln = lines[i]
        i += 1
        if ln and ln[0] != "%" and ln.split():
            raise ParseError(f"line {i}: data past the declared entry count")
    dt = np.complex128 if cplx else np.float64
    return CsrMatrix.from_triplets(rows, cols, np.array(r_l, np.int64), np.array(c_l, np.int64),
                                   np.array(v_l, dt))


def read_matrix_market(path: str) -> CsrMatrix:
    """read_matrix_market (matrix_market.cpp:91-95)."""
    with open(path) as fh:
        return parse_matrix_market(fh.read())


# ----------------------------------------------------------- seeded draws ---
def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def fill_gaussian(n: int, q: int, seed: int, stream: int) -> np.ndarray:
    """fill_gaussian (philox.hpp:92-99): column-major n x q standard normals."""
    out = np.empty((n, q), np.float64, order="F")
    check(lib().adp_fill_gaussian(_ptr(out), n, q, seed, stream))
    return out


def fill_rademacher(n: int, q: int, seed: int, stream: int) -> np.ndarray:
    """fill_rademacher (philox.hpp:102-109)."""
    out = np.empty((n, q), np.float64, order="F")
    check(lib().adp_fill_rademacher(_ptr(out), n, q, seed, stream))
    return out


def philox_uniform(seed: int, stream: int, first: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    check(lib().adp_philox_uniform(seed, stream, first, count, _ptr(out)))
    return out


def philox_gaussian(seed: int, stream: int, first: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    check(lib().adp_philox_gaussian(seed, stream, first, count, _ptr(out)))
    return out


def philox_block(seed: int, stream: int, counter: int) -> np.ndarray:
    out = np.empty(4, np.uint32)
    check(lib().adp_philox_block(seed, stream, counter, _ptr(out)))
    return out
