"""TEST INFRASTRUCTURE: numpy step backend for paper_2604_00914_b200.distributed.

Restates the fused step kernel's arithmetic (cheb_lean.cu / the reference's
maspmm + Eigen update, proj/src/cheb_filter.cpp:162-177) in numpy with the same
per-row, ascending-column accumulation order, so a gloo run of the
DistributedFilter driver on CPU is bitwise comparable with the single-process
oracle. The halo exchange goes through torch.distributed (gloo) exactly as the
CUDA backend's goes through NCCL.
"""
import random
import time

import numpy as np

FIRST, STEP, DEG1, SPMM, SPMM_ACC = 0, 1, 2, 3, 4


class NumpyStepBackend:
    def __init__(self, jitter: float = 0.0, seed: int = 0):
        # jitter: random sleeps (seconds) around the exchange points, so concurrent ranks (threads)
        # interleave in many orders -- a protocol race would show up as a wrong (non-bitwise) result
        self.jitter = jitter
        self.rng = random.Random(seed)

    def _jit(self):
        if self.jitter:
            time.sleep(self.rng.random() * self.jitter)

    def upload(self, part):
        return part.csr

    def alloc(self, n, q, cplx=False):
        return np.zeros((n, q), np.complex128 if cplx else np.float64)

    def width(self, x):
        return x.shape[1]

    def rows(self, buf, lo, hi):
        return buf[lo:hi]

    def copy_rows(self, dst, src):
        dst[...] = src

    def scale(self, x, s):
        return s * x

    def step(self, op, part, mode, g, vin, yin, out, wout, rows, s0, s1, s2, s3):
        lo, hi = rows
        rp, ci, val = op.row_ptr, op.col_idx, op.values
        nr = hi - lo
        counts = np.diff(rp[lo:hi + 1])
        kmax = int(counts.max()) if nr else 0
        acc = np.zeros((nr, g.shape[1]), g.dtype)
        for k in range(kmax):
            m = counts > k
            idx = rp[lo:hi][m] + k
            w = g[ci[idx]]
            if mode == FIRST:
                w = s2 * w
            acc[m] = acc[m] + val[idx][:, None] * w
        own = g[np.arange(lo, hi) + part.goff]
        if mode == STEP:
            t = s0 * acc
            t = t + s1 * own
            t = t - vin[lo:hi]
            out[lo:hi] = t + s2 * yin[lo:hi]
        elif mode == FIRST:
            wn = s2 * own
            wout[lo:hi] = wn
            out[lo:hi] = s0 * acc + s1 * wn
        elif mode == DEG1:
            out[lo:hi] = s0 * own + s1 * (s2 * acc + s3 * own)
        elif mode == SPMM:
            out[lo:hi] = acc
        else:
            raise ValueError(mode)

    def exchange_start(self, ops):
        import torch
        import torch.distributed as dist

        p2p = []
        for kind, peer, buf in ops:
            t = torch.from_numpy(np.ascontiguousarray(buf)) if kind == "send" else torch.from_numpy(buf)
            p2p.append(dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer))
        return dist.batch_isend_irecv(p2p)

    def exchange_wait(self, works):
        for w in works:
            w.wait()

    def synchronize(self):
        pass

    # ---- peer-memory halo (PeerHaloFilter), ranks as threads of one process --------------------
    def base(self, block):
        return block

    def new_counters(self, world):
        return np.zeros(world, np.int64)

    def step_push(self, op, part, mode, g, vin, yin, out, wout, rows, s0, s1, s2, s3, targets):
        lo, hi = rows
        self.step(op, part, mode, g, vin, yin, out, wout, rows, s0, s1, s2, s3)
        self._jit()
        for blk, tlo, thi, shift in targets:  # the kernel's epilogue stores: the rows it computed
            a, b = max(lo, tlo), min(hi, thi)
            if a < b:
                blk[a + shift:b + shift] = out[a:b]

    def push_rows(self, src, lo, hi, targets):
        for blk, tlo, thi, shift in targets:
            a, b = max(lo, tlo), min(hi, thi)
            if a < b:
                blk[a + shift:b + shift] = src[a:b]

    def signal(self, slots, value):
        self._jit()
        for c, i in slots:
            c[i] = value

    def wait(self, slots, expected, timeout_ms):
        t0 = time.time()
        for c, i in slots:
            while c[i] < expected:
                if time.time() - t0 > timeout_ms / 1e3:
                    raise TimeoutError("halo wait timed out")
                time.sleep(1e-5)
        self._jit()

    def check(self):
        pass
