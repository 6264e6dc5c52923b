#!/usr/bin/env python
"""Benchmark of the Chebyshev-filter hot path (driver contract: one JSON line on rank 0).

A "step" is one ``clenshaw_apply`` call (proj/src/cheb_filter.cpp:129-179) --
rho(l(A)) X at the configuration's initial filter degree k1 -- on config 2 of
BASELINE.json (n = 1e6 7-point Anderson Laplacian, block q = 256, fp64), the
largest single-GPU configuration the metric is quoted on.

  value  effective HBM GB/s = algorithmic bytes of the step / device time,
         inputs resident in HBM (CUDA events on the launching stream).
  e2e    the same metric through the reference-facing C-ABI call
         adp_filter_apply with pinned HOST column-major X / Y (H2D + D2H and
         the layout transposes inside the timed region).
  roofline  the fused Clenshaw-step kernel: algorithmic bytes per launch /
         average launch duration vs the measured HBM copy bandwidth.
  cpu_baseline  the CPU oracle (faithful restatement of the reference's
         maspmm + Eigen update, OpenMP over all host threads) on a bounded
         sample of degree steps of the same operator.

``--impl reference`` times the reference's CPU path (the oracle port: the
reference itself needs Eigen, absent here) with all host threads on the same
workload and prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Chebyshev-filter SpMM effective HBM GB/s (% of peak); end-to-end solve time"  # BASELINE.json metric


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--degree", type=int, default=0, help="0 = the config's initial degree k1")
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline sample length")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-solve", action="store_true", help="skip the end-to-end solve (second half of the metric)")
    p.add_argument("--no-c4", action="store_true", help="skip the short config-4 (largest single-GPU stencil) measurement")
    p.add_argument("--panel", type=int, default=0)
    p.add_argument("--variant", type=int, default=0)
    p.add_argument("--halo", default="p2p", choices=["p2p", "nccl"],
                   help="N > 1: halo rows stored by the step kernel into the neighbour's block over NVLink "
                        "(p2p, CUDA IPC) or exchanged with NCCL send/recv between steps")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def step_bytes(n, nnz, q, s=8, rp=4):
    """Algorithmic bytes of one Clenshaw degree step: A once + W, V, Y read + V write."""
    return nnz * (s + 4) + (n + 1) * rp + 4 * n * q * s


def first_bytes(n, nnz, q, s=8, rp=4):
    """First step: A + Y read + W, V write (3 blocks)."""
    return nnz * (s + 4) + (n + 1) * rp + 3 * n * q * s


def call_bytes(n, nnz, q, degree, s=8):
    if degree >= 2:
        return first_bytes(n, nnz, q, s) + (degree - 1) * step_bytes(n, nnz, q, s)
    if degree == 1:
        return nnz * (s + 4) + (n + 1) * 4 + 2 * n * q * s
    return 2 * n * q * s


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines: list[str] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------- CPU legs ---
def cpu_sample(a_csr, q: int, target_seconds: float):
    """Time degree steps of the oracle (the reference's CPU path restated) on all host threads."""
    from oracle import oracle as orc

    orc.build()
    threads = orc.max_threads()
    orc.set_threads(threads)
    oa = orc.Csr(a_csr.n_rows, a_csr.n_cols, a_csr.row_ptr, a_csr.col_idx, a_csr.values)
    t = orc.Tiled(oa, 256, 64)
    sec1, _ = orc.bench_clenshaw_steps(t, q, 1)  # includes first-touch; calibrates the sample size
    steps = max(1, min(200, int(target_seconds / max(sec1, 1e-6))))
    sec, _ = orc.bench_clenshaw_steps(t, q, steps)
    return sec, steps, threads


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2604_00914_b200 import configs

    cfg = configs.CONFIGS[args.config]
    a = cfg.operator()
    n, nnz, q = a.n_rows, a.nnz, cfg.q
    degree = args.degree or configs.filter_degree(cfg)
    b = step_bytes(n, nnz, q)
    vals, tot_steps, threads = [], 0, 1
    per = max(args.cpu_seconds / max(args.steps, 1), 2.0)
    for i in range(args.warmup + args.steps):
        sec, steps, threads = cpu_sample(a, q, per if i >= args.warmup else 1.0)
        if i >= args.warmup:
            vals.append(b * steps / sec / 1e9)
            tot_steps += steps
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(call_bytes(n, nnz, q, degree) / (v * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg.description}; clenshaw_apply degree {degree}", "n": n,
                   "nnz": nnz, "q": q, "degree": degree, "bytes_per_degree_step": b},
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{tot_steps} Clenshaw degree steps (maspmm T_i=256/T_k=64 + array update) "
                                   f"over {args.steps} timed samples; ms_per_step projects the full degree-{degree} call"},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def end_to_end_solve(adp, configs, ctx, with_cpu: bool):
    """End-to-end solve time (the metric's second half) on config 1 with the narrowed window (c1s).

    GPU: wall time of adp.solve (setup + loop, stage split). CPU: a projection -- the oracle's
    measured time per degree step (the reference's maspmm + update) x the GPU run's filter work
    (sum of degree x active width, plus the k_max x 30-probe trace estimate), labelled as such.
    """
    import torch

    cfg = configs.CONFIGS["c1s"]
    a = cfg.operator()
    da = adp.DeviceCsr(a, ctx)
    scfg = adp.SolverConfig(interval_a=cfg.window[0], interval_b=cfg.window[1], rng_seed=0)
    adp.solve(da, scfg)  # warm (workspace, handles)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = adp.solve(da, scfg)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    out = {"config": "c1s: " + cfg.description, "n": a.n_rows, "window": list(cfg.window),
           "gpu_seconds": round(gpu_s, 4), "converged": res.converged, "n_eigs": int(len(res.eigenvalues)),
           "iterations": res.iterations, "spmv_total": res.spmv_total, "avg_degree": round(res.avg_degree, 1),
           "max_residual": res.max_residual, "subspace_dim": res.subspace_dim,
           "stage_seconds": {k: round(v, 4) for k, v in vars(res.timings).items()}}
    if with_cpu:
        # columns x degree-steps of filter work in the GPU run, including the setup trace estimate
        k1 = configs.filter_degree(configs.Config("tmp", "", 0, cfg.window,
                                                  (res.bounds.lambda_min, res.bounds.lambda_max), "f64", None))
        k_max = max(k1, int(math.ceil(2.5 * k1)))
        col_steps = k_max * 30 + sum(r.degree * r.active_width for r in res.history)
        sec, steps, threads = cpu_sample(a, 64, 4.0)
        per_col_step = sec / steps / 64
        out["cpu_projected_seconds"] = round(col_steps * per_col_step, 2)
        out["cpu_projection"] = (f"oracle degree-step time ({steps} steps at q=64, {threads} threads: "
                                 f"{1e3 * sec / steps:.2f} ms) x {col_steps} column-steps of the GPU run's filter work")
    return out


# ------------------------------------------------------------- GPU arm ---
def largest_config(adp, configs, ctx, peak):
    """Config 4 (128^3 27-point stencil, q = 1024 fp64: 17.2 GB per block), a short device-resident
    clenshaw_apply after the main measurement: the cube kernel (csrc/cheb_cube.cu) on its full panels.
    Reported beside the headline, not part of it (its own operator, degree and timing)."""
    import torch

    cfg = configs.CONFIGS["c4"]
    a = cfg.operator()
    n, nnz, q = a.n_rows, a.nnz, cfg.q
    k1 = configs.filter_degree(cfg)
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, int(math.ceil(2.5 * k1)), 0.5)
    da = adp.DeviceCsr(a, ctx)
    x = torch.randn(n, q, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
    y = torch.empty_like(x)
    deg = 24
    adp.clenshaw_apply_device(f, da, x, 4, out=y)  # operator plans + workspace
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(2):
        adp.clenshaw_apply_device(f, da, x, deg, out=y)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms_launch = ev0.elapsed_time(ev1) / (2 * deg)
    b_step = step_bytes(n, nnz, q)
    gbs = b_step / (ms_launch * 1e-3) / 1e9
    da.close()
    del x, y
    torch.cuda.empty_cache()
    return {"workload": f"c4: {cfg.description}; 2 x clenshaw_apply degree {deg}, inputs resident",
            "n": n, "nnz": nnz, "q": q, "bytes_per_degree_step": b_step, "ms_per_degree_step": round(ms_launch, 4),
            "value": round(gbs, 3), "unit": "GB/s", "frac_of_hbm_peak": round(gbs / peak, 4),
            "kernel": "cheb_cube_kernel (csrc/cheb_cube.cu) on the full 64-vector panels"}


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world > 1 or os.environ.get("ADP_BENCH_FORCE_DIST") == "1":
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local
    torch.cuda.set_device(device)

    import paper_2604_00914_b200 as adp
    from paper_2604_00914_b200 import configs

    cfg = configs.CONFIGS[args.config]
    a = cfg.operator()
    n, nnz, q = a.n_rows, a.nnz, cfg.q
    k1 = configs.filter_degree(cfg)
    degree = args.degree or k1
    k_max = max(degree, int(math.ceil(2.5 * k1)))
    f = adp.build_filter(cfg.window[0], cfg.window[1], cfg.bounds, k_max, 0.5)
    if world > 1 or os.environ.get("ADP_BENCH_FORCE_DIST") == "1":
        return run_distributed(args, adp, cfg, a, f, degree, rank, world, device)

    # complex128 configurations (3, 5s): 16-byte values and block elements; the e2e, CPU-baseline and
    # solve legs are real-only, so a complex line carries the device-resident measurement alone
    cplx = cfg.dtype == "c128"
    es = 16 if cplx else 8
    if cplx:
        args.no_e2e = args.no_cpu_baseline = args.no_solve = args.no_c4 = True
    ctx = adp.Context(device)
    if args.panel:
        ctx.set_panel(args.panel)
    if args.variant:
        ctx.set_tuning(args.variant)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream)
    da = adp.DeviceCsr(a, ctx)
    x = torch.empty(n, q, dtype=torch.complex128 if cplx else torch.float64, device="cuda")
    from paper_2604_00914_b200 import _native
    import ctypes as C

    qr = 2 * q if cplx else q  # (re, im) interleaved: an n x 2q real view
    _native.check(_native.lib().adp_fill_gaussian_device(ctx.h, C.c_void_p(x.data_ptr()), n, qr, qr, 0, 0))
    y = torch.empty_like(x)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        adp.clenshaw_apply_device(f, da, x, degree, out=y)
    barrier()
    clocks = ClockSampler(device)
    clocks.start()
    launches0 = ctx.launch_count
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        adp.clenshaw_apply_device(f, da, x, degree, out=y)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    launches = ctx.launch_count - launches0
    if world > 1:
        t = torch.tensor([ms_total], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    bytes_call = call_bytes(n, nnz, q, degree, es)
    value = world * bytes_call / (ms_step * 1e-3) / 1e9
    b_step = step_bytes(n, nnz, q, es)
    launch_ms = ms_step / max(degree, 1)  # every launch of the call is one fused step kernel
    achieved = b_step / (launch_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.config}/q{q}")
        except Exception:
            traffic = None

    e2e = None
    if not args.no_e2e:
        # Reference-facing call: host column-major X (Eigen layout) in pinned memory -> adp_filter_apply.
        xh = torch.empty((q, n), dtype=torch.float64).pin_memory()  # (q, n) C-order == (n, q) column-major
        xh.copy_(x.t().cpu())
        yh = torch.empty((q, n), dtype=torch.float64).pin_memory()
        import ctypes as C

        lib = _native.lib()
        coeffs = f.coeff_array()
        cnt = C.c_int64(0)

        def e2e_call():
            _native.check(lib.adp_filter_apply(ctx.h, da.h, coeffs.ctypes.data_as(C.c_void_p), f.k_max, f.l1, f.l2,
                                               degree, C.c_void_p(xh.data_ptr()), n, n, q, 0,
                                               C.c_void_p(yh.data_ptr()), n, C.byref(cnt)))

        e2e_call()  # warm (workspace allocation)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_call()
        barrier()
        t_e2e = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([t_e2e], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            t_e2e = float(t.item())
        # sanity: the host result equals the device result of the same call
        same = bool(torch.equal(yh.t().to("cuda"), y))
        e2e = {"value": round(world * bytes_call / t_e2e / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": n * q * 8,
               "d2h_bytes_per_step": n * q * 8, "ms_per_step": round(t_e2e * 1e3, 3), "matches_device_result": same,
               "api": "adp_filter_apply (C-ABI, host column-major, pinned)"}

    solve_info = None
    if rank == 0 and not args.no_solve:
        solve_info = end_to_end_solve(adp, configs, ctx, with_cpu=(world == 1 and not args.no_cpu_baseline))

    c4 = None
    if rank == 0 and world == 1 and not args.no_c4 and args.config == "c2":
        del x, y
        torch.cuda.empty_cache()
        c4 = largest_config(adp, configs, ctx, peaks()[0])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sec, steps, threads = cpu_sample(a, q, args.cpu_seconds)
        cpu = {"value": round(b_step * steps / sec / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"{steps} Clenshaw degree steps of the same operator (oracle maspmm T_i=256/T_k=64 + "
                         f"array update, OpenMP, -O3 no -march), {sec:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128" if cplx else "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg.description}; clenshaw_apply degree {degree} "
                                   f"(k1 of window [{cfg.window[0]:.6g}, {cfg.window[1]:.6g}])",
                       "n": n, "nnz": nnz, "q": q, "degree": degree, "bytes_per_degree_step": b_step,
                       "bytes_per_step": bytes_call,
                       "l2": ("inputs larger than L2 (X, W, V blocks of %.2f GB each vs 126 MB L2)" if 3 * n * q * es > 126e6
                              else "inputs fit in L2 (X, W, V blocks of %.2f GB each; no flush: a small-config line)")
                             % (n * q * es / 1e9),
                       "parallelism": "single GPU" if world == 1 else f"replicas x{world}"},
            "pct_of_hbm_peak": round(100.0 * value / world / peak, 2),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 3), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "cheb_lean_kernel (fused Clenshaw step, csrc/cheb_lean.cu)",
                         "peak_source": peak_src,
                         "launch_ms": round(launch_ms, 5)},
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "solve": solve_info,
            "largest_config": c4,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_distributed(args, adp, cfg, a, f, degree, rank, world, device):
    """N > 1: the filter row-partitioned over the ranks (strong scaling: the operator is fixed).
    Default (--halo p2p): the step kernel stores the rows each neighbour needs straight into the
    neighbour's block over NVLink (CUDA IPC mappings) and publishes a counter; the neighbour's next
    step waits on it (PeerHaloFilter). --halo nccl: NCCL send/recv of the halo rows between steps
    while interior rows compute (DistributedFilter). If the peer-memory setup fails on a box, the
    NCCL exchange is used and the JSON line says so (paper_2604_00914_b200/distributed.py)."""
    import torch
    import torch.distributed as dist

    from paper_2604_00914_b200.distributed import CudaStepBackend, DistributedFilter, IpcPeerDirectory, PeerHaloFilter

    n, nnz, q = a.n_rows, a.nnz, cfg.q
    ctx = adp.Context(device)
    be = CudaStepBackend(ctx)
    ranges = None
    g = torch.Generator(device="cuda").manual_seed(rank)

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()

    halo = args.halo
    note = None
    df = None
    if halo == "p2p":
        try:
            df = PeerHaloFilter(a, be, rank, world, IpcPeerDirectory(), timeout_ms=30000)
            r0, r1 = df.ranges[rank]
            x = torch.randn(r1 - r0, q, dtype=torch.float64, device="cuda", generator=g)
            df.apply(f.coeffs, f.l1, f.l2, x, min(degree, 3))
            torch.cuda.synchronize()
            ok = torch.tensor([1], device="cuda")
        except Exception as e:  # pragma: no cover - depends on the box's peer access
            note = f"peer-memory halo unavailable ({type(e).__name__}: {str(e)[:160]}); NCCL exchange used"
            ok = torch.tensor([0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            halo, df = "nccl", None
            note = note or "peer-memory halo failed on another rank; NCCL exchange used"
    if df is None:
        df = DistributedFilter(a, be, rank, world, ranges)
    r0, r1 = df.ranges[rank]
    x = torch.randn(r1 - r0, q, dtype=torch.float64, device="cuda", generator=g)

    for _ in range(args.warmup):
        df.apply(f.coeffs, f.l1, f.l2, x, degree)
    barrier()
    clocks = ClockSampler(device)
    clocks.start()
    launches0 = ctx.launch_count
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record()
    for _ in range(args.steps):
        y = df.apply(f.coeffs, f.l1, f.l2, x, degree)
    ev1.record()
    barrier()
    clk = clocks.stop()
    t = torch.tensor([ev0.elapsed_time(ev1) / args.steps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    bytes_call = call_bytes(n, nnz, q, degree)
    value = bytes_call / (ms_step * 1e-3) / 1e9
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            yh = df.apply(f.coeffs, f.l1, f.l2, xh.to("cuda", non_blocking=True), degree).to("cpu")
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps], device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(bytes_call / float(te.item()) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": n * q * 8, "d2h_bytes_per_step": n * q * 8,
               "api": "DistributedFilter.apply (host tensors in/out)"}
    peak, peak_src = peaks()
    # per-GPU roofline of the step kernel: this rank's share of the algorithmic bytes per degree
    # step over the time of one degree step (interior + boundary launches)
    step_ms = ms_step / max(degree, 1)
    achieved = step_bytes(n, nnz, q) / world / (step_ms * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 3), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": None,
                         "kernel": "cheb_lean_kernel (per-GPU share, interior + boundary launches)",
                         "peak_source": peak_src, "degree_step_ms": round(step_ms, 5)},
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg.description}; clenshaw_apply degree {degree}, "
                                   f"rows partitioned over {world} GPUs, halo exchange per degree step",
                       "n": n, "nnz": nnz, "q": q, "degree": degree, "bytes_per_step": bytes_call,
                       "l2": "inputs larger than L2",
                       "parallelism": f"row-partition x{world} ("
                                      + ("halo stored by the step kernel into peer memory over NVLink" if halo == "p2p"
                                         else "NCCL halo send/recv") + ")",
                       "halo": halo, **({"halo_note": note} if note else {})},
            "pct_of_hbm_peak_per_gpu": round(100.0 * value / world / peak, 2),
            "gpu_launches": ctx.launch_count - launches0, "clocks": clk, "e2e": e2e, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
