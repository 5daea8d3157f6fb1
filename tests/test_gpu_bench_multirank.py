"""bench.py under torchrun with 2 and 4 ranks sharing one GPU (gloo process group for the
plumbing, RT_BENCH_SHARE_DEVICE): exercises the multi-rank path the driver's scaling run uses --
rt_dist_init (job id broadcast), library frame assembly on rank 0 with frames in flight,
barriers, max over ranks, e2e with downloads on rank 0 -- and checks the JSON contract."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 4])
def test_bench_ranks_one_gpu(world):
    """world 2 = the eye split (shard mode 1); world 4 = tile pairs dealt round-robin (mode 2),
    the layout of the 4- and 8-GPU scaling runs."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, RT_BENCH_SHARE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "5", "--warmup", "3", "--config", "C3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    b = lines[0]
    assert b["n_gpus"] == world and b["config"]["gather"] == "peer" and b["value"] > 0
    assert b["e2e"]["download_verified"] is True
    assert b["gpu_launches"] == 5 * 3                # per frame on rank 0: slot post, trace, completion wait
    for k in ("metric", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "dtype", "roofline",
              "clocks"):
        assert k in b
