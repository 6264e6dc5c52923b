"""Step-launch time of the filter on a configuration's operator for block widths / leading dimensions
that are not multiples of the sweep kernel's 32-column panel (the solver's active block: p = 926 on c4w).

Usage: python tools/ld_probe.py [--config c4] [--cases 1024:1024,926:926,926:928,926:960]   (q:ld pairs)
Prints ms per Step launch (degree-d call minus degree-2 call) and GB/s of algorithmic bytes at width q.
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00914_b200 as adp  # noqa: E402
from paper_2604_00914_b200 import configs  # noqa: E402
import bench  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c4")
    p.add_argument("--degree", type=int, default=42)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--cases", default="1024:1024,926:926,926:928,926:960,926:1024,420:420,420:448")
    args = p.parse_args()
    cfg = configs.CONFIGS[args.config]
    a = cfg.operator()
    n, nnz = a.n_rows, a.nnz
    k1 = configs.filter_degree(cfg)
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, max(args.degree, int(math.ceil(2.5 * k1))), 0.5)
    ctx = adp.Context(0)
    ctx.set_stream(torch.cuda.current_stream())
    da = adp.DeviceCsr(a, ctx)
    dt = torch.complex128 if a.is_complex else torch.float64
    for case in args.cases.split(","):
        q, ld = (int(t) for t in case.split(":"))
        xb = torch.randn(n, ld, dtype=dt, device="cuda")
        yb = torch.empty_like(xb)
        x, y = xb[:, :q], yb[:, :q]
        adp.clenshaw_apply_device(f, da, x, 4, out=y)
        torch.cuda.synchronize()

        def timed(deg):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                adp.clenshaw_apply_device(f, da, x, deg, out=y)
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.reps

        t2 = timed(2)
        ms = (timed(args.degree) - t2) / (args.degree - 2)
        b = bench.step_bytes(n, nnz, q, s=16 if a.is_complex else 8)
        print(f"{args.config} q={q} ld={ld} kernel={ctx.last_step_kernel}: {ms:.4f} ms/launch  {b / ms / 1e6:.1f} GB/s",
              flush=True)
        del xb, yb, x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
