import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_00914_b200 as adp
from oracle import oracle as orc
q = int(sys.argv[1])
ctx = adp.Context(0)
a = orc.random_symmetric(80, 0.1, 31)
da = adp.DeviceCsr(adp.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), ctx)
b = orc.fill_gaussian(80, q, 1, 0)
got = adp.maspmm(da, b)
print("spmm bitwise", np.array_equal(got, orc.maspmm(orc.Tiled(a, 16, 8), b)), flush=True)
