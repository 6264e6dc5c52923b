"""Complex Hermitian solves at configuration scale on one GPU (native complex128 path).

Usage:
  python tools/solve_complex.py c3 [--json out.json]          # config 3 at full size: n = 1e6, ~300 eigenpairs
  python tools/solve_complex.py c5s --width 0.1 [--json ...]  # config 5's structure at n = 2e5, generated on the
                                                              # GPU, one spectrum slice of the given width

Prints the summary, the stage split and the per-iteration history (degree, active width, Ritz values in
the window, locked count, max residual); the eigenvalues' range and the residuals are re-measured on H.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_00914_b200 as adp  # noqa: E402
from paper_2604_00914_b200 import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c3")
    ap.add_argument("--width", type=float, default=0.1, help="c5s: slice width around 0")
    ap.add_argument("--n", type=int, default=200_000, help="c5s: rows")
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    ctx = adp.Context(0)
    t0 = time.perf_counter()
    if args.config == "c3":
        cfg = configs.CONFIGS["c3"]
        h = adp.DeviceCsr(cfg.operator(), ctx)
        window, desc = cfg.window, cfg.description
    else:  # config 5's structure, generated on the device (never on the host)
        rp, ci, v = configs.random_banded_hermitian_device(args.n, 250, 20)
        h = adp.DeviceCsr.from_device(args.n, args.n, rp, ci, v, ctx)
        del rp, ci, v
        torch.cuda.empty_cache()
        window = (-args.width / 2, args.width / 2)
        desc = f"random banded Hermitian n={args.n}, half-band 250 + 20 off-band/row (config 5 structure, GPU-generated)"
    build_s = time.perf_counter() - t0
    print("operator", desc, "n", h.n_rows, "nnz", h.nnz, "window", window, f"({build_s:.1f} s)", flush=True)
    sc = adp.SolverConfig(interval_a=window[0], interval_b=window[1], rng_seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = adp.solve_hermitian(h, sc, vectors_to_host=False)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    print("seconds", round(secs, 1), "converged", r.converged, "n_eigs", len(r.eigenvalues), "iters", r.iterations,
          "p", r.subspace_dim, "e_est", round(r.e_estimate, 1), "maxres", r.max_residual, "avgdeg",
          round(r.avg_degree, 1), flush=True)
    print({k: round(v, 2) for k, v in vars(r.timings).items()})
    for it in r.history:
        print(it.iteration, it.degree, it.active_width, it.e_in_interval, it.n_locked_total, it.max_residual)
    v = r.eigenvectors
    g = (v.conj().T @ v) if len(r.eigenvalues) else None
    orth = float(torch.linalg.matrix_norm(g - torch.eye(g.shape[0], dtype=g.dtype, device=g.device)).item()) \
        if g is not None else 0.0
    out = {"config": desc, "n": h.n_rows, "nnz": h.nnz, "window": list(window), "gpu_seconds": round(secs, 2),
           "operator_seconds": round(build_s, 1), "converged": bool(r.converged), "n_eigs": len(r.eigenvalues),
           "iterations": r.iterations, "subspace_dim": r.subspace_dim, "e_estimate": r.e_estimate,
           "spmv_total": r.spmv_total, "avg_degree": r.avg_degree, "max_residual": r.max_residual,
           "tolerance": 1e-10 * max(abs(r.bounds.lambda_min), abs(r.bounds.lambda_max)),
           "bounds": [r.bounds.lambda_min, r.bounds.lambda_max], "orthonormality_fro": orth,
           "stage_seconds": vars(r.timings), "degree_history": r.degree_history,
           "eigenvalue_range": [float(np.min(r.eigenvalues)), float(np.max(r.eigenvalues))] if len(r.eigenvalues) else None,
           "solver": "solve_hermitian: native complex128 ShardedSolver on one GPU (sharded.py)"}
    print(json.dumps(out))
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
