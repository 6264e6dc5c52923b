import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_00914_b200 as adp
from oracle import oracle as orc
q = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = adp.Context(0)
a = orc.random_symmetric(80, 0.1, 31)
spec = np.linalg.eigvalsh(a.to_dense())
f = adp.build_filter(spec[10], spec[50], (spec[0] - 0.1, spec[-1] + 0.1), 60, 0.5)
g = orc.build_filter(spec[10], spec[50], (spec[0] - 0.1, spec[-1] + 0.1), 60, 0.5)
da = adp.DeviceCsr(adp.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), ctx)
x = orc.fill_gaussian(80, q, 77, 3)
for d in (0, 1, 2, 3, 25):
    try:
        got = adp.clenshaw_apply(f, da, x, d)
        want = orc.clenshaw_apply(g, orc.Tiled(a, 16, 8), x, d)
        print("q", q, "deg", d, "bitwise", np.array_equal(got, want), flush=True)
    except Exception as e:
        print("q", q, "deg", d, "ERROR", e, flush=True)
        break
try:
    b = orc.fill_gaussian(80, q, 1, 0)
    got = adp.maspmm(da, b)
    print("spmm bitwise", np.array_equal(got, orc.maspmm(orc.Tiled(a, 16, 8), b)), flush=True)
except Exception as e:
    print("spmm ERROR", e, flush=True)
