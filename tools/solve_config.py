"""Run the GPU solve on one configuration window and print the summary + iteration history.

Usage: python tools/solve_config.py [c1|c1s|c2|...] [--p P] [--json out.json]
--p sets SolverConfig.p_override (BASELINE.json's "block" size: 256 for config 2).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_00914_b200 as adp  # noqa: E402
from paper_2604_00914_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c1")
ap.add_argument("--p", type=int, default=0)
ap.add_argument("--json", default="")
args = ap.parse_args()
cfg = configs.CONFIGS[args.config]
a = cfg.operator()
ctx = adp.Context(0)
da = adp.DeviceCsr(a, ctx)
print("window", cfg.window, "bounds", cfg.bounds, "n", a.n_rows, "nnz", a.nnz, flush=True)
sc = adp.SolverConfig(interval_a=cfg.window[0], interval_b=cfg.window[1], rng_seed=0, p_override=args.p or None)
t0 = time.perf_counter()
r = adp.solve(da, sc)
torch.cuda.synchronize()
secs = time.perf_counter() - t0
print("seconds", secs, "converged", r.converged, "n_eigs", len(r.eigenvalues), "iters", r.iterations,
      "p", r.subspace_dim, "e_est", r.e_estimate, "maxres", r.max_residual, "avgdeg", r.avg_degree, flush=True)
print(vars(r.timings))
for h in r.history[:40]:
    print(h.iteration, h.degree, h.active_width, h.e_in_interval, h.n_locked_total, h.max_residual)
if args.json:
    ev = sorted(float(v) for v in r.eigenvalues)
    with open(args.json, "w") as fh:
        json.dump({"config": cfg.description, "window": list(cfg.window), "n": a.n_rows, "nnz": a.nnz,
                   "p_override": args.p or None, "gpu_seconds": round(secs, 3), "converged": bool(r.converged),
                   "n_eigs": len(ev), "iterations": r.iterations, "subspace_dim": r.subspace_dim,
                   "spmv_total": r.spmv_count if hasattr(r, "spmv_count") else None,
                   "avg_degree": r.avg_degree, "max_residual": r.max_residual, "stage_seconds": vars(r.timings),
                   "degree_history": [h.degree for h in r.history], "eigenvalue_range": [ev[0], ev[-1]] if ev else None},
                  fh, indent=1)
# python tools/solve_config.py c1  -- configs[0] as BASELINE.json states it: 40^3 7-point + U[0,1), interval 0.40-0.45 of [0, 13], GPU solve (B200)
# columns: iteration, degree, active width, Ritz values in [a, b], locked total, max residual
