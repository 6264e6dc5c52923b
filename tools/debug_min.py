import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_00914_b200 as adp
from oracle import oracle as orc
q = int(sys.argv[1]); deg = int(sys.argv[2]); variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ctx = adp.Context(0)
ctx.set_tuning(variant)
a = orc.random_symmetric(80, 0.1, 31)
f = adp.build_filter(-1.0, 1.0, (-8, 8), 60, 0.5)
da = adp.DeviceCsr(adp.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), ctx)
x = orc.fill_gaussian(80, q, 77, 3)
got = adp.clenshaw_apply(f, da, x, deg)
print("ok", q, deg, variant, float(np.abs(got).sum()), flush=True)
