"""Sample power / SM clock while a sustained clenshaw_apply_device loop runs (GPU).

Usage: python tools/power_probe.py [--config c2] [--degree 3000] [--variant 0]
Prints ms per degree step and the median power draw / SM clock during the run.
"""
import argparse
import math
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00914_b200 as adp  # noqa: E402
from paper_2604_00914_b200 import configs  # noqa: E402


def sampler(samples, stop):
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,temperature.gpu,clocks.mem",
                              "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout
        try:
            pw, sm, tc, mem = (float(v) for v in out.strip().split(","))
            samples.append((pw, sm, tc, mem))
        except ValueError:
            pass
        time.sleep(0.1)


def summarize(samples):
    s = samples[len(samples) // 4:]  # skip the ramp
    med = lambda i: sorted(v[i] for v in s)[len(s) // 2] if s else float("nan")  # noqa: E731
    return f"power {med(0):.0f} W, sm {med(1):.0f} MHz, mem {med(3):.0f} MHz, temp {med(2):.0f} C ({len(samples)} samples)"


def copy_probe(seconds):
    a = torch.empty(1 << 28, dtype=torch.float64, device="cuda").normal_()
    b = torch.empty_like(a)
    b.copy_(a)
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(samples, stop))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0, n = time.time(), 0
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(50):
            b.copy_(a)
        n += 50
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    gbs = 2 * a.numel() * 8 * n / (e0.elapsed_time(e1) * 1e6)
    print(f"copy 2 GiB: {gbs:.0f} GB/s sustained, {summarize(samples)}")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2")
    p.add_argument("--degree", type=int, default=3000)
    p.add_argument("--variant", type=int, default=0)
    p.add_argument("--panel", type=int, default=0, help="lean panel cap in columns (0 = automatic)")
    p.add_argument("--copy", type=float, default=0.0,
                   help="instead: sustained torch copy of two 2 GiB buffers for this many seconds (HBM-only reference)")
    args = p.parse_args()
    if args.copy > 0:
        return copy_probe(args.copy)
    cfg = configs.CONFIGS[args.config]
    a = cfg.operator()
    k1 = configs.filter_degree(cfg)
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, max(args.degree, int(math.ceil(2.5 * k1))), 0.5)
    ctx = adp.Context(0)
    ctx.set_stream(torch.cuda.current_stream())
    ctx.set_tuning(args.variant)
    ctx.set_panel(args.panel)
    da = adp.DeviceCsr(a, ctx)
    dt = torch.complex128 if a.is_complex else torch.float64
    x = torch.randn(a.n_rows, cfg.q, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    adp.clenshaw_apply_device(f, da, x, 50, out=y)
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(samples, stop))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    adp.clenshaw_apply_device(f, da, x, args.degree, out=y)
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / args.degree
    b_step = a.nnz * ((16 if a.is_complex else 8) + 4) + (a.n_rows + 1) * 4 + 4 * a.n_rows * cfg.q * (16 if a.is_complex else 8)
    print(f"{args.config} variant {args.variant} panel {args.panel}: {ms:.4f} ms/step, {b_step / ms / 1e6:.0f} GB/s, {summarize(samples)}")


if __name__ == "__main__":
    main()
