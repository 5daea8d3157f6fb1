"""Multi-process CPU tests of the multi-GPU host logic:
  - the library's own host protocol (rt_dist_host_selftest): shared-memory rendezvous, the
    16-slot frame-descriptor ring with flow control over more frames than slots, and the leave,
    in 2 and 3 processes -- the host half of rt_dist_init / frame renders / rt_dist_finalize;
  - world-size-2 gloo: shard map -> per-rank packed shards -> gather -> root unpack == the full
    image (the NCCL transport's data layout); max-over-ranks timing;
  - the reference arm under a 2-process launch (rank 1 exits without work)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, W, H, q):
    sys.path.insert(0, ROOT)
    from paper_1702_01530_b200 import rt
    from tests.test_abi import expected_image, synth_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    per = rt.rt_shard_bytes(W, H, world)
    mine = synth_shards(W, H, world)[rank].view(np.uint8)
    shard = torch.from_numpy(mine.copy())
    gathered = torch.zeros(world * per, dtype=torch.uint8) if rank == 0 else None
    glist = [gathered[r * per:(r + 1) * per] for r in range(world)] if rank == 0 else None
    dist.gather(shard, glist, dst=0)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = float(t[0]) == float(world)
    if rank == 0:
        L, R = rt.rt_unpack_shards_host(gathered.numpy(), W, H, world)
        got = np.stack([L, R]).view(np.uint32)[..., 0]
        ok = ok and np.array_equal(got, expected_image(W, H))
        q.put(ok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("W,H", [(93, 61), (64, 48)])
def test_gloo_world2_gather_unpack(W, H):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _selftest_worker(rank, world, job_id, frames, q, delay=0.0):
    import time
    sys.path.insert(0, ROOT)
    from paper_1702_01530_b200 import rt
    time.sleep(delay)
    q.put((rank, rt.rt_dist_host_selftest(rank, world, job_id, frames)))


def _shm_path(job_id):
    """/dev/shm file of the job's rendezvous block: FNV-1a of the 128-byte id (rt_dist.cu)."""
    h = 1469598103934665603
    for b in bytes(job_id):
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return "/dev/shm/rtb200_%016x" % h


@pytest.mark.parametrize("world", [2, 3])
def test_dist_host_protocol_multiprocess(world):
    """rt_dist_init's rendezvous + the per-frame descriptor ring (40 frames through 16 slots:
    rank 0 must wait for the slowest reader) + rt_dist_finalize's leave, in `world` processes
    with no GPU: every rank sees every frame's descriptor, in order (equal checksums)."""
    sys.path.insert(0, ROOT)
    from paper_1702_01530_b200 import rt
    job = rt.rt_dist_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_selftest_worker, args=(r, world, job, 40, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    sums = dict(q.get(timeout=10) for _ in range(world))
    assert len(set(sums.values())) == 1, sums
    # a different job id is a different rendezvous: a lone rank of a 2-world times out cleanly
    os.environ["RT_DIST_TIMEOUT_S"] = "1"
    try:
        with pytest.raises(rt.RtError) as e:
            rt.rt_dist_host_selftest(1, 2, rt.rt_dist_unique_id(), 4)
        assert e.value.status == rt.RT_ERR_PEER
    finally:
        del os.environ["RT_DIST_TIMEOUT_S"]


@pytest.mark.skipif(not os.path.isdir("/dev/shm"), reason="needs POSIX shared memory in /dev/shm")
def test_dist_peers_first_over_a_stale_empty_block():
    """Peers that start before rank 0 find a 0-byte object under the job's name (a block rank 0
    has created but not yet sized, here a stale one): they must wait until rank 0 has (re)created
    and sized it instead of mapping it (a read past the end of the object is a SIGBUS)."""
    sys.path.insert(0, ROOT)
    from paper_1702_01530_b200 import rt
    job = rt.rt_dist_unique_id()
    path = _shm_path(job)
    open(path, "wb").close()                        # 0 bytes, the state between shm_open and ftruncate
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=_selftest_worker, args=(r, 3, job, 20, q, 0.0 if r else 2.0)) for r in range(3)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0                  # -7 (SIGBUS) before the size check
        sums = dict(q.get(timeout=10) for _ in range(3))
        assert len(set(sums.values())) == 1, sums
    finally:
        if os.path.exists(path):
            os.unlink(path)


def test_reference_arm_under_torchrun():
    """`bench.py --impl reference` launched like the driver's N=2 run: rank 0 prints one JSON
    line with impl=reference, rank 1 exits 0 without work."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "C1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    ln = lines[0]
    assert ln["impl"] == "reference" and ln["n_gpus"] == 2 and ln["value"] > 0
    assert ln["e2e"]["h2d_bytes_per_step"] == 0 and ln["cpu_baseline"]["kind"] == "oracle"
