"""bench.py's N > 1 code path on one GPU: launched the way the driver launches it (torch.distributed.run,
NCCL, 127.0.0.1 rendezvous) with ONE rank and the distributed path forced (ADP_BENCH_FORCE_DIST=1), so
process-group setup, the plane-slab partition, PeerHaloFilter (no neighbours at world 1), the timing
barriers, the max-over-ranks reduction and the JSON line all run on hardware. (Ranks whose kernels wait
on one another are not emulated on one GPU; the lockstep tests cover the halo protocol.)"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("halo", ["p2p", "nccl"])
def test_bench_distributed_path_world1(halo):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, ADP_BENCH_FORCE_DIST="1")
    port = 29611 if halo == "p2p" else 29612
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "1", "--config", "c2",
           "--degree", "12", "--steps", "2", "--warmup", "3", "--halo", halo, "--e2e-steps", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{") and '"metric"' in ln]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["scaling"] == "strong"
    assert d["config"]["workload"].startswith("c2:") and d["config"]["halo"] == halo
    assert d["value"] > 100.0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert 0.0 < d["roofline"]["frac"] < 1.2
