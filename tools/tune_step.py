"""Sweep the fused-step kernel's tuning variants on one configuration (GPU).

Prints ms per Step launch (a degree-d call minus a degree-2 call, over d - 2) and
effective GB/s for each variant, and
checks that every variant's result is bitwise identical to variant 0's.
Usage: python tools/tune_step.py [--config c2] [--degree 30] [--variants 0,1,2]
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
    p.add_argument("--config", default="c2")
    p.add_argument("--degree", type=int, default=30)
    p.add_argument("--variants", default="0,2,5", help="kernel families (adp_ctx_set_tuning): 0 automatic, 1 row, "
                   "2 lean, 3 line, 4 cube, 5 sweep")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--q", type=int, default=0, help="override the block width")
    p.add_argument("--panels", default="", help="lean-kernel panel caps in columns, e.g. '128,256'")
    args = p.parse_args()
    cfg = configs.CONFIGS[args.config]
    a = cfg.operator()
    n, nnz, q = a.n_rows, a.nnz, (args.q or cfg.q)
    k1 = configs.filter_degree(cfg)
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, max(args.degree, int(math.ceil(2.5 * k1))), 0.5)
    ctx = adp.Context(0)
    ctx.set_stream(torch.cuda.current_stream())
    da = adp.DeviceCsr(a, ctx)
    g = torch.Generator(device="cuda").manual_seed(0)
    dt = torch.complex128 if a.is_complex else torch.float64
    x = torch.randn(n, q, dtype=dt, device="cuda", generator=g)
    ref = None
    b_step = bench.step_bytes(n, nnz, q, s=16 if a.is_complex else 8)
    runs = [("row", int(s), None) for s in args.variants.split(",") if s]
    for spec in filter(None, args.panels.split(",")):
        runs.append(("panel", int(spec), None))
    for kind, v, tcfg in runs:
        ctx_panel = v if kind == "panel" else 0
        ctx.set_panel(ctx_panel)
        if kind == "panel":
            v = 0
        ctx.set_tuning(v)
        y = torch.empty_like(x)
        adp.clenshaw_apply_device(f, da, x, args.degree, out=y)
        torch.cuda.synchronize()
        def timed(deg):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                adp.clenshaw_apply_device(f, da, x, deg, out=y)
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.reps

        # per Step launch: a degree-2 call (First + one Step) subtracted from the degree-d call
        t2 = timed(2)
        ms = (timed(args.degree) - t2) / (args.degree - 2)
        same = None
        if ref is None:
            ref = y.clone()
        else:
            same = bool(torch.equal(ref, y))
        label = {"row": f"variant {v}", "panel": f"lean panel cap {ctx_panel}"}[kind]
        print(f"{args.config} q={q} {label}: {ms:.4f} ms/launch  {b_step / ms / 1e6:.1f} GB/s  "
              f"bitwise_vs_first={same}", flush=True)


if __name__ == "__main__":
    main()
