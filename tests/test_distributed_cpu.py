"""Multi-process (gloo, CPU) tests of the row-partitioned Chebyshev filter driver.

world_size 2 and 3 processes run paper_2604_00914_b200.distributed.DistributedFilter
with the numpy step backend (tests/dist_numpy_backend.py) and real point-to-point
halo exchanges through torch.distributed (gloo); the gathered result must be
BITWISE equal to the single-process CPU oracle's clenshaw_apply.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _matrix(kind):
    sys.path.insert(0, ROOT)
    from paper_2604_00914_b200 import configs
    from paper_2604_00914_b200.sparse import CsrMatrix

    if kind == "lap":
        return configs.laplacian7_potential(10, -2.0, 2.0, seed=3)
    if kind == "27pt":
        return configs.dft_like_27pt(8, n_centres=4, seed=1)
    # wide band relative to the partition: halos span several ranks
    rng = np.random.default_rng(4)
    n, hb = 90, 25
    r, c = [], []
    for d in range(-hb, hb + 1):
        i = np.arange(max(0, -d), min(n, n - d))
        r.append(i)
        c.append(i + d)
    r, c = np.concatenate(r), np.concatenate(c)
    v = rng.standard_normal(len(r))
    m = CsrMatrix.from_triplets(n, n, r, c, v)
    d = m.to_dense()
    d = 0.5 * (d + d.T)
    rr, cc = np.nonzero(d)
    return CsrMatrix.from_triplets(n, n, rr, cc, d[rr, cc])


def _worker(rank, world, port, kind, degree, q, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from dist_numpy_backend import NumpyStepBackend
    from paper_2604_00914_b200.distributed import DistributedFilter
    from oracle import oracle as orc

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = _matrix(kind)
    n = a.n_rows
    ev = np.linalg.eigvalsh(a.to_dense())
    f = orc.build_filter(ev[n // 3], ev[n // 2], (ev[0] - 0.1, ev[-1] + 0.1), max(degree, 1), 0.5)
    x = orc.fill_gaussian(n, q, 9, 0)
    df = DistributedFilter(a, NumpyStepBackend(), rank, world)
    r0, r1 = df.ranges[rank]
    y = df.apply(f.coeffs, f.l1, f.l2, np.ascontiguousarray(x[r0:r1]), degree)
    np.save(f"{out_path}.{rank}.npy", np.asarray(y))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,world,degree,q", [
    ("lap", 2, 9, 6), ("lap", 2, 1, 4), ("lap", 3, 25, 5), ("27pt", 2, 12, 3), ("band", 3, 7, 2),
    ("band", 2, 2, 3), ("lap", 2, 0, 3)])
def test_distributed_filter_bitwise_vs_oracle(tmp_path, orc, kind, world, degree, q):
    import torch.multiprocessing as mp

    port = _free_port()
    out = str(tmp_path / "y")
    mp.start_processes(_worker, args=(world, port, kind, degree, q, out), nprocs=world, join=True,
                       start_method="spawn")
    a = _matrix(kind)
    n = a.n_rows
    ev = np.linalg.eigvalsh(a.to_dense())
    f = orc.build_filter(ev[n // 3], ev[n // 2], (ev[0] - 0.1, ev[-1] + 0.1), max(degree, 1), 0.5)
    x = orc.fill_gaussian(n, q, 9, 0)
    oa = orc.Csr(n, n, a.row_ptr, a.col_idx, a.values)
    want = orc.clenshaw_apply(f, orc.Tiled(oa, 256, 64), x, degree)
    got = np.concatenate([np.load(f"{out}.{r}.npy") for r in range(world)])
    assert np.array_equal(got, want)


def test_partition_and_schedule():
    sys.path.insert(0, ROOT)
    from paper_2604_00914_b200.distributed import exchange_schedule, local_part, partition_rows

    a = _matrix("lap")  # 10^3 grid: halo = one 100-row plane
    ranges = partition_rows(a, 4)
    assert ranges[0][0] == 0 and ranges[-1][1] == a.n_rows
    assert all(ranges[k][1] == ranges[k + 1][0] for k in range(3))
    parts = [local_part(a, ranges, k) for k in range(4)]
    bounds = [(p.r0, p.r1, p.cmin, p.cmax) for p in parts]
    for k, p in enumerate(parts):
        sends, recvs = exchange_schedule(bounds, k)
        # 7-point stencil on a 10^3 grid: neighbours only, one plane each way
        assert set(recvs) <= {k - 1, k + 1} and set(sends) == set(recvs)
        for peer, (lo, hi) in recvs.items():
            assert hi - lo == 100
        i0, i1 = p.interior
        assert 0 < i1 - i0 < p.n_local
        # every column of an interior row is owned
        rows = np.repeat(np.arange(p.n_local), np.diff(p.csr.row_ptr))
        cols = p.csr.col_idx + p.cmin
        sel = (rows >= i0) & (rows < i1)
        assert np.all((cols[sel] >= p.r0) & (cols[sel] < p.r1))


# ----------------------------------------------------------- peer-memory halo protocol ---
# PeerHaloFilter moves the halo inside the step (push into the neighbour's block + release
# counter; acquire wait before gathering). Here the ranks are THREADS of one process sharing
# numpy blocks, with random sleeps around every exchange point, so they really run concurrently
# and interleave in many orders: a missing wait, an early signal or a write-after-read race on
# a block's halo would make the result differ from the oracle. Two applies back to back check
# that the next filter call cannot overwrite a halo the previous one is still reading.
@pytest.mark.parametrize("kind,world,degree,q,seed", [
    ("lap", 2, 9, 6, 0), ("lap", 3, 25, 5, 1), ("lap", 4, 6, 3, 6), ("27pt", 2, 12, 3, 2), ("band", 3, 7, 2, 3),
    ("band", 2, 2, 3, 4), ("lap", 2, 1, 4, 5)])
def test_peer_halo_filter_threads_bitwise(orc, kind, world, degree, q, seed):
    import threading
    from concurrent.futures import ThreadPoolExecutor

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from dist_numpy_backend import NumpyStepBackend
    from paper_2604_00914_b200.distributed import LocalPeerDirectory, PeerHaloFilter

    a = _matrix(kind)
    n = a.n_rows
    ev = np.linalg.eigvalsh(a.to_dense())
    f = orc.build_filter(ev[n // 3], ev[n // 2], (ev[0] - 0.1, ev[-1] + 0.1), max(degree, 1), 0.5)
    xs = [orc.fill_gaussian(n, q, 9 + i, 0) for i in range(2)]
    directory = LocalPeerDirectory(threading.Barrier(world))
    filters = [PeerHaloFilter(a, NumpyStepBackend(jitter=0.002, seed=100 * seed + k), k, world, directory,
                              timeout_ms=60000) for k in range(world)]

    def rank_main(k):
        r0, r1 = filters[k].ranges[k]
        return [filters[k].apply(f.coeffs, f.l1, f.l2, np.ascontiguousarray(x[r0:r1]), degree) for x in xs]

    with ThreadPoolExecutor(world) as ex:
        res = list(ex.map(rank_main, range(world)))
    oa = orc.Csr(n, n, a.row_ptr, a.col_idx, a.values)
    for i, x in enumerate(xs):
        want = orc.clenshaw_apply(f, orc.Tiled(oa, 256, 64), x, degree)
        got = np.concatenate([res[k][i] for k in range(world)])
        assert np.array_equal(got, want), (kind, world, i)


def test_peer_halo_boundary_covers_sends_and_halo_reads():
    # the launches that push (boundary) must contain every row a neighbour needs and every row that
    # reads the halo; the interior must do neither (the write-after-read argument relies on it)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from dist_numpy_backend import NumpyStepBackend
    from paper_2604_00914_b200.distributed import LocalPeerDirectory, PeerHaloFilter

    for kind, world in (("lap", 3), ("27pt", 2), ("band", 3)):
        a = _matrix(kind)
        for k in range(world):
            pf = PeerHaloFilter(a, NumpyStepBackend(), k, world, LocalPeerDirectory())
            p = pf.part
            i0, i1 = pf.inner
            rows = np.repeat(np.arange(p.n_local), np.diff(p.csr.row_ptr))
            cols = p.csr.col_idx + p.cmin
            sel = (rows >= i0) & (rows < i1)
            assert np.all((cols[sel] >= p.r0) & (cols[sel] < p.r1))
            for lo, hi in p.sends.values():
                assert hi - p.r0 <= i0 or lo - p.r0 >= i1
            assert set(pf.neighbours) == set(p.sends) | set(p.recvs)


# A complex Hermitian operator (config 3's structure) through the peer-halo filter: blocks must be
# complex128 end to end (DistributedFilter.cplx -> backend.alloc). The numpy backend's complex
# arithmetic is its own, so the partitioned result is compared bitwise with the same backend on ONE
# rank (the partition never changes an output element's arithmetic).
@pytest.mark.parametrize("world,degree,q", [(2, 9, 3), (3, 4, 2)])
def test_peer_halo_filter_threads_complex(orc, world, degree, q):
    import threading
    from concurrent.futures import ThreadPoolExecutor

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, ROOT)
    from dist_numpy_backend import NumpyStepBackend
    from paper_2604_00914_b200 import configs
    from paper_2604_00914_b200.distributed import LocalPeerDirectory, PeerHaloFilter

    a = configs.peierls_lattice(9)
    n = a.n_rows
    f = orc.build_filter(-0.4, 0.3, (-5.0, 5.0), max(degree, 1), 0.5)
    rng = np.random.default_rng(world)
    x = rng.standard_normal((n, q)) + 1j * rng.standard_normal((n, q))

    def run(w):
        directory = LocalPeerDirectory(threading.Barrier(w))
        filters = [PeerHaloFilter(a, NumpyStepBackend(jitter=0.001, seed=k), k, w, directory, timeout_ms=60000)
                   for k in range(w)]

        def rank_main(k):
            r0, r1 = filters[k].ranges[k]
            return filters[k].apply(f.coeffs, f.l1, f.l2, np.ascontiguousarray(x[r0:r1]), degree)

        with ThreadPoolExecutor(w) as ex:
            return np.concatenate(list(ex.map(rank_main, range(w))))

    one = run(1)
    assert one.dtype == np.complex128 and np.abs(one.imag).max() > 0
    assert np.array_equal(run(world), one)
