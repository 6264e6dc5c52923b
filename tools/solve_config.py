"""Run the GPU solve on one configuration window and print the summary + iteration history.

Usage: python tools/solve_config.py [c1|c1s|...]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_00914_b200 as adp
from paper_2604_00914_b200 import configs
cfg = configs.CONFIGS[__import__("sys").argv[1] if len(__import__("sys").argv) > 1 else "c1"]
a = cfg.operator()
ctx = adp.Context(0)
da = adp.DeviceCsr(a, ctx)
print("window", cfg.window, "bounds", cfg.bounds, flush=True)
sc = adp.SolverConfig(interval_a=cfg.window[0], interval_b=cfg.window[1], rng_seed=0)
t0 = time.perf_counter()
r = adp.solve(da, sc)
torch.cuda.synchronize()
print("seconds", time.perf_counter() - t0, "converged", r.converged, "n_eigs", len(r.eigenvalues), "iters", r.iterations,
      "p", r.subspace_dim, "e_est", r.e_estimate, "maxres", r.max_residual, "avgdeg", r.avg_degree, flush=True)
print(vars(r.timings))
for h in r.history[:40]:
    print(h.iteration, h.degree, h.active_width, h.e_in_interval, h.n_locked_total, h.max_residual)
