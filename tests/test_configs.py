"""Configuration sanity: each host-built configuration's spectral bounds enclose its Gershgorin
interval, and its window lies inside the bounds.

The filter maps [lambda_min, lambda_max] onto [-1, 1] (cheb_filter.cpp:21-94); a lower bound above the
true spectrum makes the Chebyshev recurrence grow without limit at high degree (the config 4 bounds
once missed the potential wells and the trace estimate returned NaN at k_max = 765).
"""
import functools

import numpy as np
import pytest

from paper_2604_00914_b200 import configs


@functools.lru_cache(maxsize=None)
def _gershgorin(name):
    a = configs.CONFIGS[name].operator()
    rp = np.asarray(a.row_ptr, dtype=np.int64)
    ci = np.asarray(a.col_idx, dtype=np.int64)
    v = np.asarray(a.values)
    rows = np.repeat(np.arange(a.n_rows, dtype=np.int64), np.diff(rp))
    diag_mask = rows == ci
    diag = np.zeros(a.n_rows)
    np.add.at(diag, rows[diag_mask], v[diag_mask].real)
    off = np.zeros(a.n_rows)
    np.add.at(off, rows[~diag_mask], np.abs(v[~diag_mask]))
    return float((diag - off).min()), float((diag + off).max())


@pytest.mark.parametrize("name", ["c1", "c1s", "c2", "c4", "c4w"])
def test_bounds_enclose_gershgorin_and_window(name):
    cfg = configs.CONFIGS[name]
    lo, hi = _gershgorin({"c1s": "c1", "c4w": "c4"}.get(name, name))  # same operators, narrower windows
    bmin, bmax = cfg.bounds
    assert bmin <= lo and hi <= bmax, (name, (lo, hi), cfg.bounds)
    a, b = cfg.window
    assert bmin < a < b < bmax
