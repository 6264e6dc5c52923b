"""Regenerate tests/golden/*.npz (run in the build container, where /root/reference exists).

1. fixtures_*.npz: the reference's three Matrix Market test fixtures
   (/root/reference/proj/tests/fixtures/*.mtx, used by acceptance criterion 4,
   proj/tests/acceptance.cpp:210-218) converted to CSR exactly as the reference
   reader does (symmetric storage expanded, triplets sorted and duplicates
   summed: proj/src/matrix_market.cpp:22-89, csr_matrix.hpp:34-62).
2. clenshaw_golden.npz: CPU-oracle outputs of clenshaw_apply on those fixtures
   (small, so the GPU box can check against them without the oracle build).

The reference tree does not travel to the GPU box; these files do.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as orc  # noqa: E402

FIXTURES = "/root/reference/proj/tests/fixtures"
NAMES = ["laplacian2d_30", "arrow_ints", "banded_mixed"]


def read_mtx(path):
    with open(path) as fh:
        lines = fh.read().splitlines()
    sym = lines[0].split()[4].lower() == "symmetric"
    i = 1
    while lines[i].startswith("%") or not lines[i].strip():
        i += 1
    rows, cols, nnz = map(int, lines[i].split())
    r, c, v = [], [], []
    for ln in lines[i + 1:]:
        if not ln.strip() or ln.startswith("%"):
            continue
        a, b, x = ln.split()[:3]
        a, b, x = int(a) - 1, int(b) - 1, float(x)
        r.append(a); c.append(b); v.append(x)
        if sym and a != b:
            r.append(b); c.append(a); v.append(x)
    assert len([1 for ln in lines[i + 1:] if ln.strip() and not ln.startswith("%")]) == nnz
    return orc.Csr.from_triplets(rows, cols, r, c, v)


def main():
    golden = {}
    for name in NAMES:
        a = read_mtx(os.path.join(FIXTURES, name + ".mtx"))
        np.savez_compressed(os.path.join(HERE, f"fixture_{name}.npz"), n_rows=a.n_rows, n_cols=a.n_cols,
                            row_ptr=a.row_ptr, col_idx=a.col_idx, values=a.values)
        if a.n_rows != a.n_cols:
            continue
        dense = a.to_dense()
        sym = 0.5 * (dense + dense.T)
        ev = np.linalg.eigvalsh(sym)
        bounds = (ev[0] - 0.1, ev[-1] + 0.1) if np.allclose(dense, dense.T) else (
            -np.abs(dense).sum(1).max() - 0.1, np.abs(dense).sum(1).max() + 0.1)
        lo = bounds[0] + 0.3 * (bounds[1] - bounds[0])
        hi = bounds[0] + 0.45 * (bounds[1] - bounds[0])
        f = orc.build_filter(lo, hi, bounds, 40, 0.5)
        t = orc.Tiled(a, 256, 64)
        x = orc.fill_gaussian(a.n_rows, 5, 11, 0)
        for d in (0, 1, 2, 3, 17, 40):
            golden[f"{name}/deg{d}"] = orc.clenshaw_apply(f, t, x, d)
        golden[f"{name}/x"] = x
        golden[f"{name}/coeffs"] = f.coeffs
        golden[f"{name}/l1l2"] = np.array([f.l1, f.l2, f.k_max, lo, hi, bounds[0], bounds[1]])
    np.savez_compressed(os.path.join(HERE, "clenshaw_golden.npz"), **golden)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
