"""Row-sharded and complex Hermitian filtered subspace iteration (multi-GPU / complex128 solve).

The reference's ``solve`` (proj/src/solver.cpp:119-360) over a matrix whose rows are partitioned
over ``world`` ranks -- the 1-D row partition of SURVEY.md 8(e): rank k owns rows [r0, r1) of A and
of every n x p block -- for real symmetric OR complex Hermitian operators (configs 3 and 5: complex128
blocks end to end, no real 2n embedding). Per iteration and rank:

  filter          the row-partitioned Clenshaw filter (distributed.py: the fused step kernel, halo
                  rows stored into the neighbours' blocks over NVLink or exchanged with NCCL);
  CholQR2         local Gram X^H X, allreduce of the p x p Gram, replicated Cholesky with the
                  reference's shift retry (1e-14 tr / p) and rank check (1e-7), local X R^-1
                  (dense_kernels.cpp:53-92); MGS fallback with allreduced dots (:12-27);
  Rayleigh-Ritz   local A Q (halo exchange), allreduce of Q^H A Q, replicated eigh, local Q U
                  (dense_kernels.cpp:94-101);
  residuals       local |A v - lambda v|^2 column sums, allreduced (solver.cpp:94-106);
  Lanczos, trace  allreduced dots / norms (lanczos.cpp:20-111, solver.cpp:108-117);
  locking, spurious exclusion, adaptive degree: replicated host logic on O(p) scalars
                  (solver.cpp:276-332).

Random fills address the GLOBAL block (Philox fill index c * n + r, philox.hpp:96-98): a rank draws
only its rows, so every rank count sees the same initial basis, probes and top-up vectors as one
process, and the result matches the single-process solve to rounding (reduction order only). The
complex initial basis is fill_gaussian(seed, 0) + i fill_gaussian(seed, 4) (complex128 has no
reference: stream 4 is this implementation's choice); probes stay real Rademacher (Hutchinson is
exact in expectation for Hermitian f(H) with real probes).

Pluggable pieces (so the same loop runs on the GPU and, for tests, on the CPU with gloo):
  ops     dense arithmetic on local blocks: TorchOps (CUDA: cuBLAS / cuSOLVER through torch) or
          NumpyOps (CPU tests);
  sparse  filter(f, x, degree) and spmm(x) on local rows: ShardSparse (a
          DistributedFilter / PeerHaloFilter) or DeviceSparse (one GPU: the C-ABI calls);
  comm    allreduce(sum) over ranks: LocalComm, TorchComm (NCCL / gloo) or a test's ThreadComm.
"""
from __future__ import annotations

import math
import time

import numpy as np

from ._native import ConfigError
from .filter import SpectrumBounds, adaptive_degree, build_filter, initial_degree
from .solver import IterationRecord, SolveResult, SolverConfig, StageTimings
from .sparse import fill_rademacher, philox_gaussian


# ---------------------------------------------------------------------------- comms ---
class LocalComm:
    world, rank = 1, 0

    def allreduce(self, x):
        return x


class TorchComm:
    """torch.distributed all_reduce(SUM): NCCL on CUDA tensors, gloo on CPU (numpy arrays go through
    torch.from_numpy, which shares their memory)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)

    def allreduce(self, x):
        import torch

        if isinstance(x, np.ndarray):
            t = torch.from_numpy(np.ascontiguousarray(x))
            self.dist.all_reduce(t, group=self.group)
            return t.numpy()
        t = x.contiguous()
        self.dist.all_reduce(t, group=self.group)
        return t


# ------------------------------------------------------------------------- dense ops ---
class NumpyOps:
    """Local dense arithmetic on numpy arrays (CPU tests)."""

    def __init__(self, cplx: bool):
        self.cplx = cplx
        self.dt = np.complex128 if cplx else np.float64

    def from_host(self, a):
        return np.ascontiguousarray(a, self.dt)

    def host(self, a):
        return np.asarray(a)

    def zeros(self, n, p):
        return np.zeros((n, p), self.dt)

    def gram(self, x):
        return x.conj().T @ x

    def cross(self, a, b):  # a^H b
        return a.conj().T @ b

    def chol_upper(self, g):
        try:
            low = np.linalg.cholesky(g)
        except np.linalg.LinAlgError:
            return None
        r = low.conj().T
        d = np.real(np.diag(r))
        if not np.all(np.isfinite(r)) or not np.all(d > 0.0):
            return None
        return r

    def trsm_right_upper(self, x, r):  # x r^-1
        import scipy.linalg as sl

        return np.ascontiguousarray(sl.solve_triangular(r, x.T, trans="T", lower=False).T)

    def eigh(self, b):
        w, u = np.linalg.eigh(0.5 * (b + b.conj().T))
        return w, u

    def matmul(self, a, b):
        return a @ b

    def cols(self, x, idx):
        return np.ascontiguousarray(x[:, list(idx)])

    def hstack(self, blocks):
        return np.ascontiguousarray(np.concatenate(blocks, axis=1))

    def abs2_colsum(self, x):
        return np.sum(np.abs(x) ** 2, axis=0)

    def dot_re_colsum(self, a, b):
        return np.real(np.sum(a.conj() * b, axis=0))

    def diag_real(self, g):
        return np.real(np.diag(g)).copy()

    def scale_cols(self, v, lam):
        return v * np.asarray(lam, np.float64)[None, :]

    def add_diag(self, g, s):
        return g + s * np.eye(g.shape[0], dtype=g.dtype)

    def sync(self):
        pass


class TorchOps(NumpyOps):
    """Local dense arithmetic on CUDA tensors: cuBLAS GEMMs (herk / gemm / trsm) and cuSOLVER
    potrf / heevd through torch.linalg, on the current stream."""

    def __init__(self, cplx: bool, device=None):
        import torch

        self.torch = torch
        self.cplx = cplx
        self.dt = torch.complex128 if cplx else torch.float64
        self.device = device or torch.device("cuda", torch.cuda.current_device())

    def from_host(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a), device=self.device).to(self.dt)

    def host(self, a):
        return a.cpu().numpy()

    def zeros(self, n, p):
        return self.torch.zeros(n, p, dtype=self.dt, device=self.device)

    def gram(self, x):
        return x.conj().T @ x

    def cross(self, a, b):
        return a.conj().T @ b

    def chol_upper(self, g):
        t = self.torch
        low, info = t.linalg.cholesky_ex(g)
        if int(info.item()) != 0:
            return None
        r = low.mH.resolve_conj().contiguous()
        d = t.real(t.diagonal(r))
        if not bool(t.isfinite(r).all()) or not bool((d > 0.0).all()):
            return None
        return r

    def trsm_right_upper(self, x, r):
        return self.torch.linalg.solve_triangular(r, x, upper=True, left=False)

    def eigh(self, b):
        w, u = self.torch.linalg.eigh(0.5 * (b + b.conj().T))
        return w.cpu().numpy(), u

    def cols(self, x, idx):
        return x[:, self.torch.as_tensor(list(idx), dtype=self.torch.long, device=self.device)].contiguous()

    def hstack(self, blocks):
        return self.torch.cat(blocks, dim=1).contiguous()

    def abs2_colsum(self, x):
        return (x.real ** 2 + x.imag ** 2).sum(dim=0) if self.cplx else (x * x).sum(dim=0)

    def dot_re_colsum(self, a, b):
        return (a.conj() * b).real.sum(dim=0) if self.cplx else (a * b).sum(dim=0)

    def diag_real(self, g):
        return self.torch.real(self.torch.diagonal(g)).cpu().numpy().copy()

    def scale_cols(self, v, lam):
        return v * self.torch.as_tensor(np.asarray(lam, np.float64), device=self.device)[None, :]

    def add_diag(self, g, s):
        return g + s * self.torch.eye(g.shape[0], dtype=g.dtype, device=g.device)

    def sync(self):
        self.torch.cuda.synchronize()


# ---------------------------------------------------------------------------- sparse ---
def _even_ld(x):
    """A row-major CUDA block the step kernels accept and run fast on: x itself when its row pitch is
    the C-ABI's block pitch (distributed.block_ld: 16-byte vectors, whole 256-byte panels for wide
    blocks), else a copy with that layout viewed at x's width (torch.linalg may return column-major
    results; a p = 926 block's 7408-byte rows cost the sweep kernel up to 75%)."""
    if isinstance(x, np.ndarray):
        return x
    from .distributed import block_ld

    q = x.shape[1]
    if x.stride(1) == 1 and x.stride(0) == block_ld(q, x.is_complex()) and x.data_ptr() % 256 == 0:
        return x
    v = _empty_even(x)
    v.copy_(x)
    return v


def _empty_even(x):
    if isinstance(x, np.ndarray):
        return np.empty_like(x)
    import torch

    from .distributed import block_ld

    ld = block_ld(x.shape[1], x.is_complex())
    return torch.empty(x.shape[0], ld, dtype=x.dtype, device=x.device)[:, : x.shape[1]]


class ShardSparse:
    """Local rows of A over a row partition: the distributed filter and halo-exchanged SpMM."""

    def __init__(self, dfilter):
        self.f = dfilter
        self.r0, self.r1 = dfilter.ranges[dfilter.rank]

    def filter(self, f, x, degree):
        return self.f.apply(f.coeffs, f.l1, f.l2, _even_ld(x), int(degree))

    def spmm(self, x):
        return self.f.spmm(_even_ld(x))


class DeviceSparse:
    """One GPU, the whole operator: the C-ABI filter (fused step kernels) and maspmm."""

    def __init__(self, da):
        self.a = da
        self.r0, self.r1 = 0, da.n_rows

    def filter(self, f, x, degree):
        from .operator import clenshaw_apply_device

        x = _even_ld(x)
        return clenshaw_apply_device(f, self.a, x, int(degree), out=_empty_even(x))

    def spmm(self, x):
        from .operator import maspmm_device

        x = _even_ld(x)
        return maspmm_device(self.a, x, _empty_even(x), accumulate=False)


# ---------------------------------------------------------------------------- solver ---
def _wall():
    return time.perf_counter()


class ShardedSolver:
    """solve (solver.cpp:119-360) on this rank's rows [r0, r1) of an n x n operator."""

    def __init__(self, n: int, cplx: bool, ops, sparse, comm):
        self.n, self.cplx, self.ops, self.sp, self.comm = int(n), bool(cplx), ops, sparse, comm
        self.r0, self.r1 = sparse.r0, sparse.r1
        self.nl = self.r1 - self.r0
        self.spmv = 0

    # ---- global reductions
    def _sum(self, v):
        return self.comm.allreduce(v)

    def _sum_host(self, v):
        return np.asarray(self.ops.host(self._sum(v)), np.float64)

    def _norm(self, x):  # 2-norm of a distributed vector / column block (n_local x 1)
        return float(np.sqrt(self._sum_host(self.ops.abs2_colsum(x))[0]))

    # ---- global random fills: this rank's rows of the fill (index c * n + r, philox.hpp:96-98)
    def _gaussian_rows(self, seed, stream, first_col, ncols, offset=0):
        out = np.empty((self.nl, ncols))
        for j in range(ncols):
            out[:, j] = philox_gaussian(seed, stream, offset + (first_col + j) * self.n + self.r0, self.nl)
        return out

    # ---- lanczos.cpp:20-111
    def _lanczos_pass(self, steps, seed, draw_offset):
        ops = self.ops
        v = ops.from_host(philox_gaussian(seed, 1, draw_offset + self.r0, self.nl)[:, None])
        v = v * (1.0 / self._norm(v))
        basis = [v]
        alphas, betas = [], []
        scale, beta_res, breakdown = 0.0, 0.0, False
        for j in range(steps):
            bj = basis[j]
            w = self.sp.spmm(bj)
            self.spmv += 1
            alpha = float(self._sum_host(ops.dot_re_colsum(bj, w))[0])
            alphas.append(alpha)
            w = w - alpha * bj
            if j > 0:
                w = w - betas[j - 1] * basis[j - 1]
            b = ops.hstack(basis)
            for _ in range(2):  # full reorthogonalisation (lanczos.cpp:44-45)
                h = self._sum(ops.cross(b, w))
                w = w - ops.matmul(b, h)
            beta = self._norm(w)
            betas.append(beta)
            scale = max(scale, abs(alpha), beta)
            if beta <= scale * 1e-13:
                beta_res, breakdown = beta, True
                break
            if j + 1 < steps:
                basis.append(w * (1.0 / beta))
            else:
                beta_res = beta
        p = len(alphas)
        t = np.diag(alphas) + np.diag(betas[:p - 1], 1) + np.diag(betas[:p - 1], -1)
        ev, z = np.linalg.eigh(t)
        lower = ev[0] - beta_res * abs(z[p - 1, 0])
        upper = ev[-1] + beta_res * abs(z[p - 1, p - 1])
        return lower, upper, breakdown and p < steps

    def spectrum_bounds(self, steps, seed):
        n = self.n
        eff = min(steps, n)
        lower, upper = math.inf, -math.inf
        for attempt in range(4):
            lo, hi, early = self._lanczos_pass(eff, seed, attempt * n)
            lower, upper = min(lower, lo), max(upper, hi)
            if not early:
                break
        mag = max(abs(lower), abs(upper))
        if not (upper - lower > 1e-12 * mag):
            pad = max(1e-8, np.finfo(float).eps * n * mag)
            lower, upper = lower - pad, upper + pad
        return lower, upper

    # ---- solver.cpp:108-117
    def eigcount(self, f, probes, seed):
        n = self.n
        v = fill_rademacher(n, probes, seed, 2)[self.r0:self.r1] if self.nl else np.zeros((0, probes))
        vd = self.ops.from_host(v)
        w = self.sp.filter(f, vd, f.k_max)
        self.spmv += f.k_max * probes
        return float(np.sum(self._sum_host(self.ops.dot_re_colsum(vd, w)))) / probes

    # ---- dense_kernels.cpp:12-27
    def _mgs(self, x):
        ops = self.ops
        kept = []
        for j in range(x.shape[1]):
            v = ops.cols(x, [j])
            orig = self._norm(v)
            for _ in range(2):
                for q in kept:
                    c = self._sum(ops.cross(q, v))
                    v = v - ops.matmul(q, c)
            nrm = self._norm(v)
            if not (nrm > orig * 1e-13) or not (nrm > 0.0):
                continue
            kept.append(v * (1.0 / nrm))
        if not kept:
            return ops.zeros(self.nl, 0), 0
        return ops.hstack(kept), len(kept)

    # ---- dense_kernels.cpp:53-92
    def cholesky_qr(self, x):
        ops = self.ops
        p = x.shape[1]
        if p == 0:
            return x, 0
        g = self._sum(ops.gram(x))
        gd = ops.diag_real(g)
        if not np.all(np.isfinite(gd)):
            raise RuntimeError("cholesky_qr: non-finite entries")
        r = ops.chol_upper(g)
        if r is None:  # shift retry: 1e-14 * trace / p
            g = ops.add_diag(g, 1e-14 * float(np.sum(gd)) / p)
            gd = ops.diag_real(g)
            r = ops.chol_upper(g)
        if r is not None and not np.all(ops.diag_real(r) > 1e-7 * np.sqrt(gd)):  # rank check
            r = None
        if r is None:
            return self._mgs(x)
        x = ops.trsm_right_upper(x, r)
        r = ops.chol_upper(self._sum(ops.gram(x)))  # second pass (CholeskyQR2)
        if r is None:
            return self._mgs(x)
        return ops.trsm_right_upper(x, r), p

    # ---- solver.cpp:58-77
    def top_up(self, q, have, target, seed, draw_offset):
        ops = self.ops
        cols = [q] if have > 0 else []
        draw = draw_offset
        while have < target:
            v = ops.from_host(philox_gaussian(seed, 3, draw + self.r0, self.nl)[:, None])
            draw += self.n
            if have > 0:
                b = ops.hstack(cols)
                for _ in range(2):
                    h = self._sum(ops.cross(b, v))
                    v = v - ops.matmul(b, h)
            nrm = self._norm(v)
            if nrm <= 1e-8:
                continue
            cols.append(v * (1.0 / nrm))
            have += 1
        return ops.hstack(cols)

    # ---- dense_kernels.cpp:94-101
    def rayleigh_ritz(self, q):
        ops = self.ops
        aq = self.sp.spmm(q)
        b = self._sum(ops.cross(q, aq))
        w, u = ops.eigh(b)
        return np.asarray(w, np.float64), ops.matmul(q, u)

    # ---- solver.cpp:94-106
    def residuals(self, v, lam):
        ops = self.ops
        if v.shape[1] == 0:
            return np.zeros(0)
        av = self.sp.spmm(v)
        r = self._sum_host(ops.abs2_colsum(av - ops.scale_cols(v, lam)))
        self.spmv += v.shape[1]
        return np.sqrt(r)

    def solve(self, cfg: SolverConfig) -> SolveResult:
        ops, n = self.ops, self.n
        lo, hi = cfg.interval_a, cfg.interval_b
        timings = StageTimings()
        t_setup = _wall()
        lmin, lmax = self.spectrum_bounds(cfg.lanczos_steps, cfg.rng_seed)
        if not (lmin <= lo and hi <= lmax):
            raise ConfigError(f"solve: target interval lies outside the estimated spectrum [{lmin}, {lmax}]")
        a_norm = max(abs(lmin), abs(lmax))
        span = lmax - lmin
        l1, l2 = 2.0 / span, -(lmax + lmin) / span

        def mapc(x):
            return min(max(l1 * x + l2, -1.0), 1.0)

        alpha, beta = math.acos(mapc(lo)), math.acos(mapc(hi))
        k1 = initial_degree(alpha, beta, cfg.c)
        k_max = max(k1, int(math.ceil(cfg.k_multiplier * k1)))
        f = build_filter(lo, hi, (lmin, lmax), k_max, cfg.m)
        e_est = self.eigcount(f, cfg.trace_probes, cfg.rng_seed)
        bounds = SpectrumBounds(lmin, lmax)

        def result(vals, vecs, converged, iterations, history, degs, max_res, p):
            avg = float(np.mean(degs)) if degs else 0.0
            return SolveResult(np.asarray(vals, np.float64), vecs, converged, False, iterations, self.spmv, avg,
                               max_res, list(degs), history, bounds, e_est, p, timings)

        if cfg.p_override:
            p = int(cfg.p_override)
        else:
            if e_est < 0.5:
                timings.setup = _wall() - t_setup
                return result([], ops.zeros(self.nl, 0), True, 0, [], [], 0.0, 0)
            e_ceil = int(math.ceil(max(e_est, 0.0)))
            p = max(int(math.ceil(cfg.mu * e_ceil)), e_ceil + 5, 10)
        if p >= n:
            raise ConfigError("sharded solve: the subspace (p >= n) needs the dense fallback: use the one-device solve")

        x = self._gaussian_rows(cfg.rng_seed, 0, 0, p)
        xd = ops.from_host(x + 1j * self._gaussian_rows(cfg.rng_seed, 4, 0, p)) if self.cplx else ops.from_host(x)
        active, kept = self.cholesky_qr(xd)
        if kept < p:
            active = self.top_up(active, kept, p, cfg.rng_seed, 0)
        degree = min(k1, k_max)
        n_lock, n_check_prev, iteration = 0, 0, 0
        locked = ops.zeros(self.nl, 0)
        locked_values, history, degs = [], [], []
        timings.setup = _wall() - t_setup
        empty_streak, converged = 0, False
        while iteration < cfg.max_iter:
            iteration += 1
            qa = p - n_lock
            rec = IterationRecord(iteration, degree, qa, 0, n_lock, 0.0, 0, 0, -1.0)
            t = _wall()
            filtered = self.sp.filter(f, active, degree)
            rec.spmv_filter = degree * qa
            self.spmv += degree * qa
            ops.sync()
            timings.filter += _wall() - t

            t = _wall()
            stacked = ops.hstack([locked, filtered]) if n_lock else filtered
            stacked, kept = self.cholesky_qr(stacked)
            if kept < p:
                stacked = self.top_up(stacked, kept, p, cfg.rng_seed, iteration << 32)
            ops.sync()
            timings.orth += _wall() - t

            t = _wall()
            ritz, active = self.rayleigh_ritz(ops.cols(stacked, range(n_lock, p)))
            ops.sync()
            timings.rayleigh_ritz += _wall() - t

            t = _wall()
            in_iv = [j for j in range(qa) if lo <= ritz[j] <= hi]
            e_i = len(in_iv)
            rec.e_in_interval, rec.n_locked_total = e_i, n_lock
            if e_i == 0:
                empty_streak += 1
                degs.append(degree)
                history.append(rec)
                timings.other += _wall() - t
                if iteration > 3 and empty_streak >= 10:
                    converged = True
                    break
                continue
            empty_streak = 0
            next_degree = adaptive_degree(f, ritz, e_i, cfg.tau_a)
            timings.other += _wall() - t

            t = _wall()
            values_in = [float(ritz[j]) for j in in_iv]
            resid = self.residuals(ops.cols(active, in_iv), values_in)
            rec.spmv_residual = e_i
            rec.max_residual = float(np.max(resid))
            timings.residuals += _wall() - t

            t = _wall()
            tau_s = min(min(x_ - lo, hi - x_) for x_ in values_in)  # spurious_threshold (solver.cpp:81-92)
            test_set = list(range(e_i))
            if cfg.spurious_detection and tau_s > 0.0:
                checked = [c for c in range(e_i) if resid[c] < tau_s]
                n_check = len(checked) + n_lock
                if n_check > 0 and n_check == n_check_prev:
                    test_set = checked
                n_check_prev = n_check
            thr = cfg.tau_c * a_norm
            lock_cols, n_unconv = [], 0
            for c in test_set:
                if resid[c] < thr:
                    lock_cols.append(in_iv[c])
                    locked_values.append(float(ritz[in_iv[c]]))
                else:
                    n_unconv += 1
            if lock_cols:
                locked = ops.hstack([locked, ops.cols(active, lock_cols)]) if n_lock else ops.cols(active, lock_cols)
                keep = [j for j in range(qa) if j not in set(lock_cols)]
                active = ops.cols(active, keep)
            n_lock += len(lock_cols)
            rec.n_locked_total = n_lock
            degs.append(degree)
            history.append(rec)
            degree = next_degree
            timings.other += _wall() - t
            if n_unconv == 0:
                converged = True
                break

        # assemble: ascending pairs, re-measured residuals (solver.cpp:346-359)
        order = np.argsort(np.asarray(locked_values), kind="stable")
        vals = np.asarray(locked_values)[order]
        vecs = ops.cols(locked, order.tolist()) if n_lock else locked
        max_res = 0.0
        if n_lock:
            max_res = float(np.max(self.residuals(vecs, vals)))
        return result(vals, vecs, converged, iteration, history, degs, max_res, p)


def solve_sharded(a_global, cfg: SolverConfig, *, comm=None, backend="cuda", ranges=None, peer=True, ctx=None,
                  dfilter=None):
    """solve on a row partition over torch.distributed (world = comm.world; world 1 = one device).

    a_global: the host CsrMatrix (every rank builds its local rows from it); real symmetric or
    complex Hermitian. backend "cuda": this rank's GPU (the fused filter with the halo pushed over
    NVLink when ``peer``, else NCCL send/recv); "numpy": the CPU step backend (tests). Returns this
    rank's SolveResult; its eigenvectors are this rank's rows [r0, r1).
    """
    comm = comm or (TorchComm() if _dist_ready() else LocalComm())
    cplx = bool(a_global.is_complex)
    if dfilter is None and comm.world == 1 and backend == "cuda":
        from .operator import DeviceCsr, default_context

        import torch

        da = DeviceCsr(a_global, ctx or default_context(torch.cuda.current_device()))
        return ShardedSolver(a_global.n_rows, cplx, TorchOps(cplx), DeviceSparse(da), comm).solve(cfg)
    if dfilter is None:
        from .distributed import CudaStepBackend, DistributedFilter, IpcPeerDirectory, PeerHaloFilter

        be = CudaStepBackend(ctx)
        if peer and comm.world > 1:
            dfilter = PeerHaloFilter(a_global, be, comm.rank, comm.world, IpcPeerDirectory(), ranges=ranges)
        else:
            dfilter = DistributedFilter(a_global, be, comm.rank, comm.world, ranges)
    ops = NumpyOps(cplx) if backend == "numpy" else TorchOps(cplx)
    return ShardedSolver(a_global.n_rows, cplx, ops, ShardSparse(dfilter), comm).solve(cfg)


def _dist_ready() -> bool:
    try:
        import torch.distributed as dist

        return dist.is_available() and dist.is_initialized()
    except Exception:
        return False
