"""Multi-GPU row partition of the Chebyshev filter with per-degree halo exchange.

The reference is single-process; the paper only describes a
row-partitioned MPI layout. Here one process drives one GPU:

* rank k owns a contiguous row range [r0, r1) of A and of the n x q blocks;
* its CSR keeps only those rows, with columns re-indexed into a halo-extended
  local layout  [halo_lo | own rows | halo_hi]  covering [cmin, cmax] (the
  contiguous superset of the columns the rows touch -- exact for banded and
  stencil operators); own row r sits at local row r + goff, goff = r0 - cmin;
* the Clenshaw recurrence (proj/src/cheb_filter.cpp:162-177) runs step by step:
  before each degree step the boundary rows of the current W that neighbours
  need are exchanged (point-to-point send/recv through torch.distributed: NCCL
  over NVLink on GPUs, gloo on CPU), while the INTERIOR rows -- whose columns
  are all local -- are computed on the compute stream; the boundary rows are
  computed once the halo has landed;
* every rank's arithmetic is the single-GPU kernel's, in the same per-row
  order, so the gathered distributed result is bitwise identical to the
  single-process result (tests/test_distributed_cpu.py, tests/test_gpu_parity.py).

The per-step kernel comes from a backend: ``CudaStepBackend`` (the C-ABI
``adp_step_device`` on torch CUDA tensors) in the product; the CPU test suite
plugs in a numpy restatement of the same step to exercise this driver under
gloo.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .sparse import CsrMatrix

FIRST, STEP, DEG1, SPMM, SPMM_ACC = 0, 1, 2, 3, 4


def partition_rows(a: CsrMatrix, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges balancing nonzeros + rows (the step streams both)."""
    n = a.n_rows
    work = np.diff(a.row_ptr).astype(np.float64) + 1.0
    csum = np.concatenate([[0.0], np.cumsum(work)])
    cuts = [0]
    for k in range(1, world):
        cuts.append(int(np.searchsorted(csum, csum[-1] * k / world)))
    cuts.append(n)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


@dataclass
class LocalPart:
    """Rank-local slice of A with its halo layout and exchange schedule."""

    rank: int
    world: int
    r0: int
    r1: int
    cmin: int
    cmax: int
    csr: CsrMatrix  # local rows, columns re-indexed to cmin-based local rows
    interior: tuple[int, int]  # local row range whose columns are all owned
    sends: dict = field(default_factory=dict)  # peer -> (global lo, hi) of MY rows the peer needs
    recvs: dict = field(default_factory=dict)  # peer -> (global lo, hi) of peer rows I need

    @property
    def goff(self) -> int:
        return self.r0 - self.cmin

    @property
    def n_local(self) -> int:
        return self.r1 - self.r0

    @property
    def n_ext(self) -> int:
        return self.cmax - self.cmin + 1


def local_part(a: CsrMatrix, ranges, rank: int) -> LocalPart:
    r0, r1 = ranges[rank]
    rp = a.row_ptr[r0:r1 + 1] - a.row_ptr[r0]
    cols = a.col_idx[a.row_ptr[r0]:a.row_ptr[r1]]
    vals = a.values[a.row_ptr[r0]:a.row_ptr[r1]]
    cmin = int(min(cols.min(), r0)) if len(cols) else r0
    cmax = int(max(cols.max(), r1 - 1)) if len(cols) else r1 - 1
    csr = CsrMatrix(r1 - r0, cmax - cmin + 1, rp.astype(np.int64), (cols - cmin).astype(np.int64), vals.copy())
    # interior rows: all columns inside [r0, r1)
    rows = np.repeat(np.arange(r1 - r0), np.diff(rp))
    outside = (cols < r0) | (cols >= r1)
    bad = np.zeros(r1 - r0, bool)
    bad[rows[outside]] = True
    good = np.flatnonzero(~bad)
    # largest contiguous interior block (stencils: everything but one plane on each side)
    if len(good):
        runs = np.split(good, np.flatnonzero(np.diff(good) != 1) + 1)
        best = max(runs, key=len)
        interior = (int(best[0]), int(best[-1]) + 1)
    else:
        interior = (0, 0)
    part = LocalPart(rank, len(ranges), r0, r1, cmin, cmax, csr, interior)
    return part


def exchange_schedule(parts_bounds: list[tuple[int, int, int, int]], rank: int):
    """parts_bounds[k] = (r0, r1, cmin, cmax) of every rank -> (sends, recvs) of `rank`."""
    r0, r1, cmin, cmax = parts_bounds[rank]
    sends, recvs = {}, {}
    for peer, (p0, p1, pmin, pmax) in enumerate(parts_bounds):
        if peer == rank:
            continue
        lo, hi = max(p0, cmin), min(p1, cmax + 1)  # peer rows I need
        if lo < hi:
            recvs[peer] = (lo, hi)
        lo, hi = max(r0, pmin), min(r1, pmax + 1)  # my rows the peer needs
        if lo < hi:
            sends[peer] = (lo, hi)
    return sends, recvs


class DistributedFilter:
    """clenshaw_apply over a row partition: Y_local = rho(l(A)) X restricted to my rows.

    ``backend`` provides: alloc(n_rows, q) -> block, rows(block, lo, hi) -> view,
    copy_rows(dst, src), step(part, mode, g, vin, yin, out, wout, rows, s0..s3),
    scale(dst, src, s), exchange(ops) and synchronize().
    """

    def __init__(self, a_global: CsrMatrix, backend, rank: int, world: int, ranges=None):
        self.world, self.rank = world, rank
        self.ranges = ranges or partition_rows(a_global, world)
        self.part = local_part(a_global, self.ranges, rank)
        self.cplx = bool(a_global.is_complex)  # blocks are complex128 for a complex operator
        bounds = []
        for k in range(world):
            p0, p1 = self.ranges[k]
            cols = a_global.col_idx[a_global.row_ptr[p0]:a_global.row_ptr[p1]]
            bounds.append((p0, p1, int(min(cols.min(), p0)) if len(cols) else p0,
                           int(max(cols.max(), p1 - 1)) if len(cols) else p1 - 1))
        self.part.sends, self.part.recvs = exchange_schedule(bounds, rank)
        self.backend = backend
        self.op = backend.upload(self.part)

    # rows of the halo-extended layout
    def _ext(self, glo, ghi):
        return glo - self.part.cmin, ghi - self.part.cmin

    def _halo(self, buf):
        ops = []
        for peer, (lo, hi) in self.part.sends.items():
            a, b = self._ext(lo, hi)
            ops.append(("send", peer, self.backend.rows(buf, a, b)))
        for peer, (lo, hi) in self.part.recvs.items():
            a, b = self._ext(lo, hi)
            ops.append(("recv", peer, self.backend.rows(buf, a, b)))
        return ops

    def _run(self, mode, g, vin, yin, out, wout, s):
        """One degree step: exchange g's halo while interior rows compute, then the boundary."""
        part, be = self.part, self.backend
        pending = be.exchange_start(self._halo(g)) if part.sends or part.recvs else None
        i0, i1 = part.interior
        if i1 > i0:
            be.step(self.op, part, mode, g, vin, yin, out, wout, (i0, i1), *s)
        if pending is not None:
            be.exchange_wait(pending)
        for lo, hi in ((0, i0), (i1, part.n_local)):
            if hi > lo:
                be.step(self.op, part, mode, g, vin, yin, out, wout, (lo, hi), *s)

    def spmm(self, x_local):
        """My rows of A X (maspmm, tiled_matrix.hpp:184-210): X's halo rows exchanged, then the Spmm
        mode of the step kernel (the sharded solve's Rayleigh-Ritz, residuals and Lanczos)."""
        be, part = self.backend, self.part
        q = be.width(x_local)
        ext = be.alloc(part.n_ext, q, self.cplx)
        g0, g1 = part.goff, part.goff + part.n_local
        be.copy_rows(be.rows(ext, g0, g1), x_local)
        out = be.alloc(part.n_local, q, self.cplx)
        self._run(SPMM, ext, None, None, out, None, (0.0, 0.0, 0.0, 0.0))
        return out

    def apply(self, coeffs, l1, l2, x_local, degree: int):
        """x_local: my n_local x q rows (backend block). Returns my rows of rho(l(A)) X."""
        be, part = self.backend, self.part
        deg = int(degree)
        while deg > 0 and coeffs[deg] == 0.0:  # cheb_filter.cpp:141-142
            deg -= 1
        q = be.width(x_local)
        if deg == 0:
            return be.scale(x_local, float(coeffs[0]))
        n_ext = part.n_ext
        a_buf, b_buf = be.alloc(n_ext, q, self.cplx), be.alloc(n_ext, q, self.cplx)
        g0, g1 = part.goff, part.goff + part.n_local
        if deg == 1:
            be.copy_rows(be.rows(a_buf, g0, g1), x_local)
            out = be.alloc(part.n_local, q, self.cplx)
            self._run(DEG1, a_buf, None, None, out, None, (coeffs[0], coeffs[1], l1, l2))
            return out
        # the First step gathers Y: Y needs its halo too, so stage it in an extended buffer
        y_ext = be.alloc(n_ext, q, self.cplx)
        be.copy_rows(be.rows(y_ext, g0, g1), x_local)
        # w = c_d y -> a_buf ; v -> b_buf
        self._run(FIRST, y_ext, None, None, be.rows(b_buf, g0, g1), be.rows(a_buf, g0, g1),
                  (2.0 * l1, 2.0 * l2 + coeffs[deg - 1] / coeffs[deg], coeffs[deg], 0.0))
        cur_w, cur_v = b_buf, a_buf
        for j in range(deg - 2, 0, -1):
            v_rows = be.rows(cur_v, g0, g1)
            self._run(STEP, cur_w, v_rows, x_local, v_rows, None, (2.0 * l1, 2.0 * l2, coeffs[j], 0.0))
            cur_w, cur_v = cur_v, cur_w
        out = be.alloc(part.n_local, q, self.cplx)
        self._run(STEP, cur_w, be.rows(cur_v, g0, g1), x_local, out, None, (l1, l2, coeffs[0], 0.0))
        return out


def block_ld(q: int, cplx: bool = False) -> int:
    """Leading dimension (elements) of a row-major device block of q columns, as csrc/capi.cu block_ld:
    an even number of fp64 columns, and whole 256-byte panels for blocks wider than one panel."""
    m = 16 if cplx else 32
    if q > m:
        return (q + m - 1) // m * m
    return q if cplx else ((q + 1) // 2) * 2


class CudaStepBackend:
    """Device backend: torch CUDA tensors + adp_step_device; halo via torch.distributed (NCCL)."""

    def __init__(self, ctx=None):
        import torch

        from .operator import default_context

        self.torch = torch
        self.ctx = ctx or default_context(torch.cuda.current_device())

    def upload(self, part: LocalPart):
        from .operator import DeviceCsr

        return DeviceCsr(part.csr, self.ctx)

    def alloc(self, n, q, cplx=False):
        # row pitch as the C-ABI's own blocks (block_ld): 16-byte aligned rows, whole 256-byte panels
        # once the block is wider than one (misaligned rows cost the sweep kernel 15-75%)
        ld = block_ld(q, cplx)
        dt = self.torch.complex128 if cplx else self.torch.float64
        return self.torch.zeros(n, ld, dtype=dt, device="cuda")[:, :q]

    def width(self, x):
        return x.shape[1]

    def rows(self, buf, lo, hi):
        return buf[lo:hi]

    def copy_rows(self, dst, src):
        dst.copy_(src)

    def scale(self, x, s):
        return x * s

    def step(self, op, part, mode, g, vin, yin, out, wout, rows, s0, s1, s2, s3):
        import ctypes as C

        from ._native import check, lib

        t = self.torch
        self.ctx.set_stream(t.cuda.current_stream())
        lo, hi = rows
        ptr = lambda x: C.c_void_p(x.data_ptr()) if x is not None else C.c_void_p(0)  # noqa: E731
        q = g.shape[1]
        ld_y = yin.stride(0) if yin is not None else g.stride(0)
        ld_out = out.stride(0)
        check(lib().adp_step_device(self.ctx.h, op.h, mode, ptr(g), g.stride(0), ptr(vin), ptr(yin), ld_y,
                                    ptr(out), ptr(wout), ld_out, q, lo, hi, part.goff, s0, s1, s2, s3))

    def exchange_start(self, ops):
        import torch.distributed as dist

        p2p, landing = [], []
        for kind, peer, buf in ops:
            if kind == "send":
                p2p.append(dist.P2POp(dist.isend, buf.contiguous(), peer))
            else:  # NCCL needs contiguous receive buffers: land, then scatter into the strided rows
                tmp = buf if buf.is_contiguous() else self.torch.empty(buf.shape, dtype=buf.dtype, device=buf.device)
                p2p.append(dist.P2POp(dist.irecv, tmp, peer))
                if tmp is not buf:
                    landing.append((buf, tmp))
        return dist.batch_isend_irecv(p2p), landing

    def exchange_wait(self, pending):
        works, landing = pending
        for w in works:
            w.wait()
        for view, tmp in landing:
            view.copy_(tmp)

    def synchronize(self):
        self.torch.cuda.synchronize()

    # ---- peer-memory halo (PeerHaloFilter) ----------------------------------------------------
    def base(self, block):
        """The full-width allocation behind a block view (what is published to the neighbours)."""
        return block._base if block._base is not None else block

    def new_counters(self, world: int):
        c = self.torch.zeros(world, dtype=self.torch.int64, device="cuda")
        self.torch.cuda.synchronize()
        return c

    def _halo_targets(self, targets):
        from ._native import HaloTarget

        arr = (HaloTarget * max(1, len(targets)))()
        for i, (blk, lo, hi, shift) in enumerate(targets):
            arr[i] = HaloTarget(blk.data_ptr(), lo, hi, shift, blk.stride(0))
        return arr, len(targets)

    def step_push(self, op, part, mode, g, vin, yin, out, wout, rows, s0, s1, s2, s3, targets):
        import ctypes as C

        from ._native import check, lib

        t = self.torch
        self.ctx.set_stream(t.cuda.current_stream())
        lo, hi = rows
        ptr = lambda x: C.c_void_p(x.data_ptr()) if x is not None else C.c_void_p(0)  # noqa: E731
        arr, n = self._halo_targets(targets)
        ld_y = yin.stride(0) if yin is not None else g.stride(0)
        check(lib().adp_step_device_push(self.ctx.h, op.h, mode, ptr(g), g.stride(0), ptr(vin), ptr(yin), ld_y,
                                         ptr(out), ptr(wout), out.stride(0), g.shape[1], lo, hi, part.goff,
                                         s0, s1, s2, s3, arr, n))

    def push_rows(self, src, lo, hi, targets):
        import ctypes as C

        from ._native import check, lib

        self.ctx.set_stream(self.torch.cuda.current_stream())
        arr, n = self._halo_targets(targets)
        from ._native import ADP_C128, ADP_F64

        dt = ADP_C128 if src.is_complex() else ADP_F64
        check(lib().adp_halo_push_rows(self.ctx.h, dt, C.c_void_p(src.data_ptr()), src.stride(0), lo, hi, src.shape[1],
                                       arr, n))

    def signal(self, slots, value: int):
        import ctypes as C

        from ._native import check, lib

        self.ctx.set_stream(self.torch.cuda.current_stream())
        ptrs = (C.c_void_p * len(slots))(*[c.data_ptr() + 8 * i for c, i in slots])
        check(lib().adp_halo_signal(self.ctx.h, ptrs, len(slots), int(value)))

    def wait(self, slots, expected: int, timeout_ms: int):
        import ctypes as C

        from ._native import check, lib

        self.ctx.set_stream(self.torch.cuda.current_stream())
        ptrs = (C.c_void_p * len(slots))(*[c.data_ptr() + 8 * i for c, i in slots])
        check(lib().adp_halo_wait(self.ctx.h, ptrs, len(slots), int(expected), int(timeout_ms)))

    def check(self):
        from ._native import check, lib

        check(lib().adp_halo_check(self.ctx.h))


# ---------------------------------------------------------------------------------------------
# Peer-memory halo: the step kernel itself moves the halo (no separate collective)
# ---------------------------------------------------------------------------------------------
class LocalPeerDirectory:
    """Peer buffers of ranks that live in ONE process (emulated ranks, threads): a rank's registered
    arrays are visible to the others as they are. With a barrier (threads), publish waits for all."""

    def __init__(self, barrier=None):
        self.buffers = {}
        self.barrier = barrier

    def publish(self, rank: int, items: dict):
        for name, t in items.items():
            self.buffers[(rank, name)] = t
        if self.barrier is not None:
            self.barrier.wait()
        return items

    def lookup(self, rank: int, name: str):
        return self.buffers[(rank, name)]


class IpcPeerDirectory:
    """Peer buffers across processes, one GPU each: tensors are exported with torch's CUDA IPC
    reduction (cudaIpcGetMemHandle of the allocation + offset), exchanged with all_gather_object and
    mapped into this process (cudaIpcOpenMemHandle: NVLink peer memory between GPUs)."""

    def __init__(self, group=None):
        self.group = group
        self.buffers = {}

    def publish(self, rank: int, items: dict):
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        mine = {name: reduce_tensor(t) for name, t in items.items()}
        world = dist.get_world_size(self.group)
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, mine), group=self.group)
        for peer, exported in gathered:
            if peer == rank:
                continue
            for name, (fn, args) in exported.items():
                self.buffers[(peer, name)] = fn(*args)
        return items

    def lookup(self, rank: int, name: str):
        return self.buffers[(rank, name)]


class PeerHaloFilter(DistributedFilter):
    """clenshaw_apply over a row partition with the halo exchange FUSED into the step kernel.

    Each rank's halo-extended blocks (Y, W, V) and a counter array are published to its
    neighbours (CUDA IPC: NVLink peer memory). Per degree step, on the compute stream:
      wait   -- until every neighbour's counter reaches this step's epoch: the halo of the block
                being gathered has landed (adp_halo_wait, acquire / system scope);
      boundary rows (the rows that read the halo or that a neighbour needs) -- the step kernel
                stores each output row a neighbour needs straight into that neighbour's halo of the
                same block, from the epilogue that computed it (adp_step_device_push);
      signal -- publish the epoch to every neighbour (adp_halo_signal, release / system scope);
      interior rows -- local only; they overlap the neighbours' consumption of the pushed rows.
    The signal follows ALL boundary work (also on the last step, and the next call's first push
    waits for it), so a neighbour's next push into a block's halo waits until this rank has
    finished gathering from it (no write-after-read race); neighbours are the union of senders
    and receivers, so the counters are symmetric. Every rank's arithmetic is
    the single-GPU kernel's: the gathered result is bitwise identical to one device.

    ``backend`` adds to DistributedFilter's interface: step_push(op, part, mode, g, vin, yin, out,
    wout, rows, s0..s3, targets), push_rows(src, lo, hi, targets), new_counters(world),
    signal(counter_slots, value), wait(counter_slots, expected, timeout_ms) and check();
    a target is (peer block, row_lo, row_hi, row_shift). ``CudaStepBackend`` is the product;
    apply_steps() yields after every exchange point so tests can run emulated ranks in lockstep.
    """

    def __init__(self, a_global: CsrMatrix, backend, rank: int, world: int, directory, ranges=None,
                 timeout_ms: int = 60000):
        super().__init__(a_global, backend, rank, world, ranges)
        self.directory = directory
        self.timeout_ms = int(timeout_ms)
        self.bounds = []
        for k in range(world):
            p0, p1 = self.ranges[k]
            cols = a_global.col_idx[a_global.row_ptr[p0]:a_global.row_ptr[p1]]
            self.bounds.append((p0, p1, int(min(cols.min(), p0)) if len(cols) else p0,
                                int(max(cols.max(), p1 - 1)) if len(cols) else p1 - 1))
        part = self.part
        self.neighbours = sorted(set(part.sends) | set(part.recvs))
        # interior rows: read no halo AND are sent to nobody (pushes happen in boundary launches only)
        i0, i1 = part.interior
        for lo, hi in part.sends.values():
            lo, hi = lo - part.r0, hi - part.r0
            if hi <= i0 or lo >= i1:
                continue
            if lo - i0 < i1 - hi:
                i0 = max(i0, hi)
            else:
                i1 = min(i1, lo)
        self.inner = (i0, max(i0, i1))
        self.q = None
        self.epoch = 0

    def _prepare(self, q: int):
        """Blocks of width q and the counters, published to the neighbours (collective when over IPC)."""
        if self.q == q:
            return
        be, part = self.backend, self.part
        self.bufs = {name: be.alloc(part.n_ext, q, self.cplx) for name in ("y", "a", "b")}
        self.counters = be.new_counters(self.world)
        items = {f"buf_{k}": be.base(v) for k, v in self.bufs.items()}
        items["counters"] = self.counters
        self.directory.publish(self.rank, items)
        self.peer_bufs = self.peer_counters = None  # resolved after every rank has published
        self.q = q
        self.epoch = 0

    def _resolve(self):
        if self.peer_bufs is None:
            self.peer_bufs = {p: {k: self.directory.lookup(p, f"buf_{k}") for k in self.bufs} for p in self.neighbours}
            self.peer_counters = {p: self.directory.lookup(p, "counters") for p in self.neighbours}

    def _targets(self, name: str):
        """My rows each neighbour needs -> its rows of block `name`: (block, lo, hi, shift) in my local rows."""
        part = self.part
        return [(self.peer_bufs[peer][name], lo - part.r0, hi - part.r0, part.r0 - self.bounds[peer][2])
                for peer, (lo, hi) in part.sends.items()]

    def _signal(self):
        self.epoch += 1
        self.backend.signal([(self.peer_counters[p], self.rank) for p in self.neighbours], self.epoch)

    def _wait(self):
        self.backend.wait([(self.counters, p) for p in self.neighbours], self.epoch, self.timeout_ms)

    def _step(self, mode, g, vin, yin, out, wout, rows, s, push_name):
        if rows[1] <= rows[0]:
            return
        if push_name is None or not self.part.sends:
            return self.backend.step(self.op, self.part, mode, g, vin, yin, out, wout, rows, *s)
        self.backend.step_push(self.op, self.part, mode, g, vin, yin, out, wout, rows, *s, self._targets(push_name))

    def _run_fused(self, mode, g, vin, yin, out, wout, s, push_name):
        part = self.part
        i0, i1 = self.inner
        if self.neighbours:
            self._wait()
        for rows in ((0, i0), (i1, part.n_local)):
            self._step(mode, g, vin, yin, out, wout, rows, s, push_name)
        if self.neighbours:  # after the last step too: "done gathering from my halos" for the next call
            self._signal()
        self._step(mode, g, vin, yin, out, wout, (i0, i1), s, None)

    def _push_input(self, x_local, name: str):
        """Own rows of the filter's input into the neighbours' halo of block `name` (rows already computed).
        Waits first for the neighbours' last signal of the previous call: they no longer read that halo."""
        if self.neighbours and self.epoch > 0:
            self._wait()
        if self.part.sends:
            self.backend.push_rows(x_local, 0, self.part.n_local, self._targets(name))
        if self.neighbours:
            self._signal()

    def apply_steps(self, coeffs, l1, l2, x_local, degree: int):
        """Generator form of apply(): yields after each exchange point; its return value is the result."""
        be, part = self.backend, self.part
        deg = int(degree)
        while deg > 0 and coeffs[deg] == 0.0:  # cheb_filter.cpp:141-142
            deg -= 1
        q = be.width(x_local)
        if deg == 0:
            return be.scale(x_local, float(coeffs[0]))
        fresh = self.q != q
        self._prepare(q)
        if fresh:
            yield  # every rank publishes its blocks before anyone maps a neighbour's
        self._resolve()
        g0, g1 = part.goff, part.goff + part.n_local
        y_ext, a_buf, b_buf = self.bufs["y"], self.bufs["a"], self.bufs["b"]
        if deg == 1:
            be.copy_rows(be.rows(a_buf, g0, g1), x_local)
            self._push_input(x_local, "a")
            yield
            out = be.alloc(part.n_local, q, self.cplx)
            self._run_fused(DEG1, a_buf, None, None, out, None, (coeffs[0], coeffs[1], l1, l2), None)
            be.check()
            return out
        be.copy_rows(be.rows(y_ext, g0, g1), x_local)
        self._push_input(x_local, "y")
        yield
        # w = c_d y -> a ; v -> b (pushed: the next step gathers b)
        self._run_fused(FIRST, y_ext, None, None, be.rows(b_buf, g0, g1), be.rows(a_buf, g0, g1),
                        (2.0 * l1, 2.0 * l2 + coeffs[deg - 1] / coeffs[deg], coeffs[deg], 0.0), "b")
        yield
        cur_w, cur_v, names = b_buf, a_buf, ("b", "a")
        for j in range(deg - 2, 0, -1):
            v_rows = be.rows(cur_v, g0, g1)
            self._run_fused(STEP, cur_w, v_rows, x_local, v_rows, None, (2.0 * l1, 2.0 * l2, coeffs[j], 0.0), names[1])
            yield
            cur_w, cur_v, names = cur_v, cur_w, (names[1], names[0])
        out = be.alloc(part.n_local, q, self.cplx)
        self._run_fused(STEP, cur_w, be.rows(cur_v, g0, g1), x_local, out, None, (l1, l2, coeffs[0], 0.0), None)
        be.check()
        return out

    def apply(self, coeffs, l1, l2, x_local, degree: int):
        gen = self.apply_steps(coeffs, l1, l2, x_local, degree)
        while True:
            try:
                next(gen)
            except StopIteration as stop:
                return stop.value


def run_lockstep(filters, xs, coeffs, l1, l2, degree):
    """Drive several ranks' PeerHaloFilter.apply_steps round-robin, one exchange point at a time, on
    ONE stream: every wait is already satisfied when it is queued (its signal was queued earlier),
    so no kernel ever waits on a concurrently running one. Returns each rank's result."""
    gens = [f.apply_steps(coeffs, l1, l2, x, degree) for f, x in zip(filters, xs)]
    out = [None] * len(gens)
    live = set(range(len(gens)))
    while live:
        for k in sorted(live):
            try:
                next(gens[k])
            except StopIteration as stop:
                out[k] = stop.value
                live.discard(k)
    return out
