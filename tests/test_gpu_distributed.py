"""Row-partitioned filter on the GPU, ranks emulated as threads on ONE device.

Each emulated rank runs DistributedFilter with the CUDA step backend (the
product kernel, adp_step_device) on its own context and stream; halo rows move
through a host-side mailbox (the only change versus the NCCL exchange). No
kernel ever waits on another rank's kernel (B200_PROFILING.md forbids that on
one GPU): the exchange is host-synchronised. The gathered result must be
bitwise equal to the single-GPU clenshaw_apply.
"""
import threading

import numpy as np
import pytest

import paper_2604_00914_b200 as adp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


class Mailbox:
    def __init__(self):
        self.cv = threading.Condition()
        self.msgs = {}

    def post(self, key, value):
        with self.cv:
            self.msgs[key] = value
            self.cv.notify_all()

    def take(self, key):
        with self.cv:
            while key not in self.msgs:
                self.cv.wait(timeout=60)
            return self.msgs.pop(key)


def make_backend(mailbox, rank):
    from paper_2604_00914_b200.distributed import CudaStepBackend

    class ThreadBackend(CudaStepBackend):
        def __init__(self):
            super().__init__(adp.Context(0))
            self.calls = 0
            self.stream = torch.cuda.Stream()

        def exchange_start(self, ops):
            self.calls += 1
            # clone on this rank's stream and FINISH before posting: the receiver copies on its own stream
            # and must not overtake the clone (seen at 128^3: 60 MB halo planes)
            clones = [(peer, buf.clone()) for kind, peer, buf in ops if kind == "send"]
            torch.cuda.current_stream().synchronize()
            for peer, c in clones:
                mailbox.post((rank, peer, self.calls), c)
            return [(buf, (peer, rank, self.calls)) for kind, peer, buf in ops if kind == "recv"]

        def exchange_wait(self, pending):
            # the posted clone lives in the SENDER's stream pool of the caching allocator: finish the copy
            # before dropping the last reference, or the sender may reuse the memory while this rank's
            # stream still reads it (seen as corrupted halo planes on 64^3 grids; NCCL's own exchange
            # records the streams itself)
            for buf, key in pending:
                src = mailbox.take(key)
                buf.copy_(src)
                torch.cuda.current_stream().synchronize()
                del src

    return ThreadBackend()


def run_ranks(a, world, fn):
    mailbox = Mailbox()
    results, errors = [None] * world, []

    def body(rank):
        try:
            be = make_backend(mailbox, rank)
            with torch.cuda.stream(be.stream):
                results[rank] = fn(rank, be)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    if errors:
        raise errors[0]
    return results


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,degree,q,kind", [(2, 12, 64, "lap"), (3, 7, 6, "lap"), (2, 1, 130, "lap"),
                                                  (4, 20, 256, "lap"),
                                                  # slabs of whole grid planes (bench.py --gpus N --halo nccl, and
                                                  # solve_sharded without peer memory): the plane-sweep kernel on the
                                                  # interior slab and on the one-plane boundary launches
                                                  (2, 12, 64, "lap_planes"), (4, 9, 100, "lap_planes"),
                                                  (2, 8, 64, "27pt_planes"), (3, 11, 40, "27pt_planes"),
                                                  # more (panel, tile) items than SMs: every persistent CTA of the
                                                  # sweep kernel walks several items of a RANGED launch
                                                  (2, 5, 64, "27pt40_planes"), (2, 5, 256, "27pt40_planes"),
                                                  (3, 4, 117, "27pt40_planes"), (2, 6, 256, "lap40_planes"),
                                                  (2, 5, 117, "27pt64_planes"), (2, 3, 128, "27pt64_planes")])
def test_emulated_ranks_bitwise(orc, world, degree, q, kind):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    from paper_2604_00914_b200 import configs
    from paper_2604_00914_b200.distributed import DistributedFilter

    import re

    m = re.search(r"(\d+)_planes", kind)
    if kind.startswith("lap"):
        nx = int(m.group(1)) if m else 20
        a, plane = configs.laplacian7_potential(nx, -2.0, 2.0, seed=1), nx * nx
        f = adp.build_filter(5.9, 6.1, (-2.0, 14.0), 40, 0.5)
    else:
        nx = int(m.group(1)) if m else 12
        a, plane = configs.dft_like_27pt(nx, 4, 2), nx * nx
        f = adp.build_filter(0.2, 0.6, (-5.9, 8.6), 40, 0.5)
    ranges = bench.plane_ranges(a.n_rows, plane, world) if kind.endswith("_planes") else None
    n = a.n_rows
    x = orc.fill_gaussian(n, q, 3, 0)
    want = adp.clenshaw_apply(f, adp.DeviceCsr(a), x, degree)
    kernels = [None] * world

    def fn(rank, be):
        df = DistributedFilter(a, be, rank, world, ranges)
        r0, r1 = df.ranges[rank]
        xl = be.alloc(r1 - r0, q)  # the backend's block pitch (odd widths need the pad column)
        xl.copy_(torch.from_numpy(np.ascontiguousarray(x[r0:r1])))
        out = df.apply(f.coeffs, f.l1, f.l2, xl, degree).cpu().numpy()
        kernels[rank] = be.ctx.last_step_kernel
        return out

    got = np.concatenate(run_ranks(a, world, fn))
    assert np.array_equal(got, want)
    if ranges is not None and degree >= 2:
        assert all(k == 5 for k in kernels), kernels  # every rank's Step launches took the plane-sweep kernel


# ------------------------------------------------ halo pushed by the step kernel (peer memory) ---
# PeerHaloFilter with the product backend: the lean kernel's epilogue stores the rows a neighbour
# needs straight into the neighbour's block (here: another emulated rank's tensor on the same
# device; across GPUs the same store goes over NVLink to a CUDA-IPC mapping), and the 1-thread
# signal / wait kernels order the exchange. The emulated ranks share ONE stream and run in
# lockstep (run_lockstep): every wait is queued after the signal it waits for, so no kernel
# waits on a concurrently running one. Bitwise equal to the single-device filter; two calls
# back to back, ragged and narrow widths (narrow ones push with the copy kernel).
@pytest.mark.parametrize("world,degree,q,kind", [(2, 12, 64, "lap"), (3, 7, 6, "lap"), (2, 1, 130, "lap"),
                                                  (4, 20, 256, "lap"), (2, 9, 2, "lap"), (3, 5, 100, "27pt"),
                                                  (2, 6, 256, "27pt"),  # interior rows: cube kernel, ranged plan
                                                  (2, 8, 5, "herm"), (3, 5, 64, "herm"),  # complex128 blocks
                                                  # slabs of whole grid planes: the plane-sweep kernel on the
                                                  # interior AND on the pushed boundary planes
                                                  (2, 12, 64, "lap_planes"), (3, 9, 40, "27pt_planes"),
                                                  (4, 6, 34, "27pt_planes"),
                                                  # more (panel, tile) items than SMs on the interior slabs AND on
                                                  # the one-plane push launches (the multi-GPU bench's shape:
                                                  # config 4 has 8192 items per launch)
                                                  (2, 5, 256, "27pt40_planes"), (3, 4, 200, "lap40_planes")])
def test_peer_halo_lockstep_bitwise(orc, world, degree, q, kind):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_00914_b200 import configs
    from paper_2604_00914_b200.distributed import CudaStepBackend, LocalPeerDirectory, PeerHaloFilter, run_lockstep

    ranges = None
    if kind == "herm":  # config 3's structure: complex128 blocks through alloc, steps and pushes
        a = configs.peierls_lattice(24)
    else:
        big = "40" in kind
        a = (configs.laplacian7_potential(40 if big else 20, -2.0, 2.0, seed=1) if kind.startswith("lap")
             else configs.dft_like_27pt(40 if big else 12, 4, 2))
    if kind.endswith("_planes"):
        import bench

        plane = (1600 if big else 400) if kind.startswith("lap") else (1600 if big else 144)
        ranges = bench.plane_ranges(a.n_rows, plane, world)
    n = a.n_rows
    f = adp.build_filter(5.9, 6.1, (-2.0, 14.0), 40, 0.5) if kind != "herm" else adp.build_filter(-0.3, 0.2, (-5.0, 5.0), 40, 0.5)
    ctx = adp.Context(0)
    ctx.set_stream(torch.cuda.current_stream())
    directory = LocalPeerDirectory()
    filters = [PeerHaloFilter(a, CudaStepBackend(ctx), k, world, directory, ranges=ranges, timeout_ms=5000)
               for k in range(world)]
    launches0 = ctx.launch_count
    for seed in (3, 4):
        x = orc.fill_gaussian(n, q, seed, 0)
        if kind == "herm":
            x = x + 1j * orc.fill_gaussian(n, q, seed + 10, 0)
        want = adp.clenshaw_apply(f, adp.DeviceCsr(a, ctx), x, degree)
        xs = []
        for k in range(world):
            r0, r1 = filters[k].ranges[k]
            xs.append(torch.from_numpy(np.ascontiguousarray(x[r0:r1])).cuda())
        outs = run_lockstep(filters, xs, f.coeffs, f.l1, f.l2, degree)
        got = np.concatenate([o.cpu().numpy() for o in outs])
        assert np.array_equal(got, want), seed
        if ranges is not None:
            assert ctx.last_step_kernel == 5
    assert ctx.launch_count > launches0


def _ipc_worker(rank, port, out_path):
    import os
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    import paper_2604_00914_b200 as adp
    from paper_2604_00914_b200.distributed import CudaStepBackend, IpcPeerDirectory
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    ctx = adp.Context(0)
    be = CudaStepBackend(ctx)
    q, n_ext = 40, 64
    blk = be.alloc(n_ext, q)
    counters = be.new_counters(2)
    d = IpcPeerDirectory()
    d.publish(rank, {"blk": be.base(blk), "counters": counters})
    peer = 1 - rank
    pblk, pcnt = d.lookup(peer, "blk"), d.lookup(peer, "counters")
    src = torch.arange(10 * q, dtype=torch.float64, device="cuda").reshape(10, q) + 1000.0 * rank
    # rows 3..7 of mine land at the peer's rows 3 + 20 + rank ... (shift 20 + rank); then the counter
    be.push_rows(src, 0, 10, [(pblk, 3, 8, 20 + rank)])
    be.signal([(pcnt, rank)], 7 + rank)
    torch.cuda.synchronize()
    dist.barrier()  # host-side: no kernel waits on the other process
    ok_rows = torch.equal(blk[3 + 20 + peer:8 + 20 + peer], (torch.arange(10 * q, dtype=torch.float64, device="cuda")
                                                           .reshape(10, q) + 1000.0 * peer)[3:8])
    untouched = float(blk.abs().sum()) == float(blk[3 + 20 + peer:8 + 20 + peer].abs().sum())
    with open(f"{out_path}.{rank}", "w") as fh:
        fh.write(f"{int(ok_rows)} {int(untouched)} {int(counters[peer])}\n")
    # teardown order: drop the peer's imported mappings, then wait until BOTH processes have done so
    # before either exits (an exporter leaving while its peer still maps its memory can kill the peer)
    del pblk, pcnt, d
    import gc

    gc.collect()
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


def test_ipc_directory_push_and_signal_two_processes(tmp_path):
    # the cross-process half of the peer-memory halo: torch CUDA IPC export / import of a block and
    # the counters (IpcPeerDirectory), rows stored into the other process's block at the right
    # shift, the counter value published. Two processes on the one device; neither kernel waits.
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "ipc")
    mp.start_processes(_ipc_worker, args=(port, out), nprocs=2, join=True, start_method="spawn")
    for rank in range(2):
        ok_rows, untouched, cnt = open(f"{out}.{rank}").read().split()
        assert ok_rows == "1" and untouched == "1" and int(cnt) == 7 + (1 - rank)
