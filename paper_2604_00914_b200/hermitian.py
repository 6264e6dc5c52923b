"""Eigenpairs of complex Hermitian operators (configs 3 and 5), natively in complex128 on the device.

The reference solver is real symmetric only (``solve`` in proj/src/solver.cpp:119-360
takes a CsrMatrixd). ``solve_hermitian`` runs the same filtered subspace iteration on H itself
(sharded.ShardedSolver with complex128 blocks on one GPU): the complex fused filter kernel, complex
SpMM, Gram matrices X^H X and projections Q^H A Q through cuBLAS zgemm / zherk-class products,
Cholesky (zpotrf) and the Hermitian eigensolver (zheevd) through cuSOLVER, residuals on H. No host
numpy arithmetic and no real 2n embedding in the product path.

``hermitian_embedding`` (the real 2n x 2n S = [[A, -B], [B, A]] of H = A + iB, whose spectrum is H's
with doubled multiplicity) stays as a TEST PIN: it ties the complex path to the real, reference-exact
one (tests/test_oracle_pins.py, tests/test_gpu_solver.py).
"""
from __future__ import annotations

import numpy as np

from .solver import SolveResult, SolverConfig
from .sparse import CsrMatrix


def hermitian_embedding(h: CsrMatrix) -> CsrMatrix:
    """The real 2n x 2n embedding S of a complex Hermitian CSR matrix H (structural zeros dropped).

    Row r of S holds (c, Re h_rc) and (c + n, -Im h_rc); row r + n holds (c, Im h_rc) and
    (c + n, Re h_rc). Columns stay strictly ascending per row (all c < n <= c' + n).
    """
    if h.n_rows != h.n_cols:
        raise ValueError("hermitian_embedding: square matrices only")
    n = h.n_rows
    rp = np.asarray(h.row_ptr, np.int64)
    ci = np.asarray(h.col_idx, np.int64)
    v = np.asarray(h.values, np.complex128)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    re, im = v.real, v.imag
    blocks = [(rows, ci, re), (rows, ci + n, -im), (rows + n, ci, im), (rows + n, ci + n, re)]
    r = np.concatenate([b[0] for b in blocks])
    c = np.concatenate([b[1] for b in blocks])
    x = np.concatenate([b[2] for b in blocks])
    keep = x != 0.0
    return CsrMatrix.from_triplets(2 * n, 2 * n, r[keep], c[keep], x[keep])


def solve_hermitian(h, config: SolverConfig, ctx=None, vectors_to_host: bool = True) -> SolveResult:
    """Interior eigenpairs of a complex Hermitian operator in [interval_a, interval_b] on this process's
    GPU (torch's current device unless ``ctx`` is given). ``h``: a host CsrMatrix or a complex DeviceCsr
    (config 5's operator is generated on the device and never exists on the host)."""
    import torch

    from .operator import DeviceCsr, default_context
    from .sharded import DeviceSparse, LocalComm, ShardedSolver, TorchOps

    if not h.is_complex:
        raise ValueError("solve_hermitian: complex operator expected (use solve for real symmetric ones)")
    if h.n_rows != h.n_cols:
        raise ValueError("solve_hermitian: square operators only")
    if isinstance(h, DeviceCsr):
        da, own = h, False
    else:
        ctx = ctx or default_context(torch.cuda.current_device())
        da, own = DeviceCsr(h, ctx), True
    try:
        ops = TorchOps(True, torch.device("cuda", da.ctx.device))
        r = ShardedSolver(h.n_rows, True, ops, DeviceSparse(da), LocalComm()).solve(config)
    finally:
        if own:
            da.close()
    if vectors_to_host:
        r.eigenvectors = r.eigenvectors.cpu().numpy() if hasattr(r.eigenvectors, "cpu") else r.eigenvectors
    return r
