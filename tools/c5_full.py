"""Config 5 at FULL size on one GPU (n = 4e6, half-band 250 + 20 off-band/row, ~2.16 G nonzeros, complex128).

The operator is generated on the device (configs.random_banded_hermitian_device), uploaded with
adp_csr_create_device (int64 row offsets: nnz >= 2^31), and one spectrum slice's filter is timed:
clenshaw_apply on a q = 384 complex128 block at the slice's initial degree would take hours, so a
bounded number of degree steps is timed (CUDA events on the launching stream) and reported per step,
with SM clocks sampled during the timed region.

Usage: python tools/c5_full.py [--degree 8] [--q 384] [--out gpurun_out/c5_full.json]
Config 5 is FP64-issue bound: the kernel does 4 DMUL + 4 DADD per complex
multiply-accumulate (no FMA: bitwise parity with the reference's SSE2 arithmetic), so the
roofline reported is FP64 instructions against the unfused FP64 issue peak (half the DFMA flop peak).
"""
import argparse
import json
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00914_b200 as adp  # noqa: E402
from paper_2604_00914_b200 import configs  # noqa: E402
import bench  # noqa: E402

FP64_DFMA_TFLOPS = bench.fp64_peak()[0]  # measured DFMA peak (profiles/fp64_peak.json), FMA = 2 flops


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--degree", type=int, default=8)
    p.add_argument("--q", type=int, default=384)
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--out", default="gpurun_out/c5_full.json")
    p.add_argument("--variant", type=int, default=0, help="kernel family (0 automatic: band-block kernel)")
    p.add_argument("--n", type=int, default=4_000_000, help="rows (config 5: 4e6)")
    args = p.parse_args()
    cfg = configs.CONFIGS["c5"]
    ctx = adp.Context(0)
    ctx.set_stream(torch.cuda.current_stream())
    ctx.set_tuning(args.variant)
    t0 = time.time()
    rp, ci, v = configs.random_banded_hermitian_device(args.n, 250, 20)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    n, nnz = rp.numel() - 1, ci.numel()
    t0 = time.time()
    da = adp.DeviceCsr.from_device(n, n, rp, ci, v, ctx)
    del rp, ci, v
    torch.cuda.empty_cache()
    upload_s = time.time() - t0
    # spectral radius by power iteration on one vector (a lower estimate; the map uses cfg.bounds)
    x1 = torch.randn(n, 1, dtype=torch.complex128, device="cuda")
    y1 = torch.empty_like(x1)
    rad = 0.0
    for _ in range(30):
        x1 /= torch.linalg.vector_norm(x1)
        adp.maspmm_device(da, x1, y1, accumulate=False)
        rad = float(torch.linalg.vector_norm(y1))
        x1, y1 = y1, x1
    del x1, y1
    k1 = configs.filter_degree(cfg)
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, max(args.degree, int(math.ceil(2.5 * k1))), 0.5)
    q = args.q
    x = torch.randn(n, q, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    adp.clenshaw_apply_device(f, da, x, 2, out=y)  # warm-up (allocates the W / V workspace)
    torch.cuda.synchronize()
    clocks = bench.ClockSampler(0)
    clocks.start()
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        adp.clenshaw_apply_device(f, da, x, args.degree, out=y)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / args.degree)
    clk = clocks.stop()
    ms = min(times)
    b_step = nnz * (16 + 4) + (n + 1) * 8 + 4 * n * q * 16
    flops = 8 * nnz * q + 12 * n * q
    tflops = flops / ms / 1e9
    peak_gbs, peak_src = bench.peaks()
    out = {
        "config": cfg.description,
        "n": n,
        "nnz": nnz,
        "nnz_per_row": nnz / n,
        "row_offsets": "int64 (nnz >= 2^31)",
        "q": q,
        "degree_steps_timed": args.degree,
        "ms_per_degree_step": round(ms, 3),
        "ms_per_step_all_reps": [round(t, 3) for t in times],
        "initial_degree_k1": k1,
        "projected_filter_seconds_at_k1": round(ms * k1 / 1e3, 1),
        "bytes_per_step": b_step,
        "effective_gbs": round(b_step / ms / 1e6, 1),
        "hbm_frac": round(b_step / ms / 1e6 / peak_gbs, 4),
        "hbm_peak": [peak_gbs, peak_src],
        "flops_per_step": flops,
        "fp64_tflops": round(tflops, 2),
        "fp64_frac_of_dfma_peak": round(tflops / FP64_DFMA_TFLOPS, 4),
        "step_kernel": ctx.last_step_kernel,
        "spectral_radius_power_iteration": round(rad, 3),
        "bounds_used": list(cfg.bounds),
        "window": list(cfg.window),
        "generate_seconds": round(gen_s, 1),
        "upload_seconds": round(upload_s, 1),
        "gpu_mem_peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
        "clocks": clk,
    }
    line = json.dumps(out)
    print(line)
    if args.out:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
