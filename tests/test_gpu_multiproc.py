"""Fused render -> gather on one GPU with two processes: rank 1 maps rank 0's framebuffers with
CUDA IPC and its trace kernel stores its tiles into them (RT_RENDER_PEER_STORE); the assembled
stereo frame must equal a single-process render bit-exactly (SURVEY §4 T3 invariant).
Same-device IPC exercises exactly the code path NVLink peers use (mapped peer pointers)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1702_01530_b200 import multigpu, rt, scenes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = scenes.scene_c2().with_view(width=93, height=61, max_depth=3)
    R = rt.StereoRenderer(0)
    R.upload(s)
    R.set_camera(s.rig)
    # three small framebuffer slots (frames in flight): they share caching-allocator blocks, so
    # several mappings of one IPC handle at different offsets
    fbs = [R.alloc_fb(s.width, s.height) for _ in range(3)]
    for fb in fbs:
        fb.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    frames = [multigpu.PeerFrame(R, fb, rank, world, dist, s.width, s.height) for fb in fbs]
    streams = [torch.cuda.Stream() for _ in fbs]
    for f, st in zip(frames, streams):
        f.render(s.max_depth, st)
    torch.cuda.synchronize()
    frames[0].assemble()
    if rank == 0:
        ref = R.render(s.width, s.height, s.max_depth)["fb"]
        torch.cuda.synchronize()
        q.put(all(bool(torch.equal(ref, fb)) for fb in fbs))
    dist.barrier()
    for f in frames:
        f.close()
    R.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_store_frame_bit_exact(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
