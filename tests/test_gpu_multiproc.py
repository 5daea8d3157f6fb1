"""Multi-GPU frames through the C ABI (rt_dist_init) with 2 and 3 processes on
one GPU: every rank renders its tiles of each frame and the library assembles the frame in rank
0's framebuffers -- peer stores into rank 0's IPC-mapped framebuffers, ordered by device-side
flags (same-device IPC exercises exactly the code path NVLink peers use).  Frames are kept in
flight on 3 streams per rank, more frames than the 16-slot descriptor ring, each frame with its
own camera; every assembled frame must equal the single-process render bit for bit.
Python only broadcasts the job id; no torch.distributed data-path call is made."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_FRAMES = 20


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, transport, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1702_01530_b200 import multigpu, rt, scenes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = scenes.scene_c3().with_view(width=93, height=61, max_depth=3)
    R = rt.StereoRenderer(0)
    R.upload(s)
    rigs = [scenes.c5_rig(10 * k) for k in range(5)]
    info = multigpu.join_world(R, rank, world, dist, transport)
    ok = info["world"] == world and info["rank"] == rank
    streams = [torch.cuda.Stream() for _ in range(3)]
    fbs = []
    for k in range(N_FRAMES):
        fb = R.alloc_fb(s.width, s.height) if rank == 0 else None
        if fb is not None:
            fb.zero_()
            streams[k % 3].wait_stream(torch.cuda.current_stream())
        fbs.append(fb)
        R.set_camera(rigs[k % len(rigs)])
        multigpu.Frame(R, fb, s.width, s.height).render(s.max_depth, streams[k % 3])
    torch.cuda.synchronize()
    info = rt.rt_dist_info(R.ctx)
    ok = ok and info["frames"] == N_FRAMES
    rt.rt_dist_finalize(R.ctx)
    if rank == 0:
        ref = []
        for rg in rigs:
            R.set_camera(rg)
            ref.append(R.render(s.width, s.height, s.max_depth)["fb"])
        torch.cuda.synchronize()
        bad = [k for k in range(N_FRAMES) if not torch.equal(fbs[k], ref[k % len(rigs)])]
        q.put((ok and not bad, info["transport"], bad))
    dist.barrier()
    R.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_frames_bit_exact(world):
    """world 2 = the eye split (rank 1 stores the whole right eye into rank 0's FB); world 3 =
    tile pairs dealt round-robin."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "peer", q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    ok, transport, bad = q.get(timeout=10)
    assert transport == "peer"
    assert ok, f"frames differing from the single-GPU render: {bad}"


def test_nccl_transport_one_rank():
    """The NCCL transport's whole data path on one GPU (NCCL refuses two ranks on one device): a
    one-rank world joined with RT_DIST_NCCL packs its tiles into the shard ring, runs a one-rank
    ncclGather and unpacks on the root; 20 frames in flight on 3 streams with changing cameras,
    RGBA8 and RGBA16F, must equal the local render bit for bit."""
    import sys
    sys.path.insert(0, ROOT)
    from paper_1702_01530_b200 import multigpu, rt, scenes
    s = scenes.scene_c3().with_view(width=93, height=61, max_depth=3)
    R = rt.StereoRenderer(0)
    R.upload(s)
    rigs = [scenes.c5_rig(10 * k) for k in range(5)]
    try:
        rt.rt_dist_init(R.ctx, 0, 1, rt.rt_dist_unique_id(), rt.RT_DIST_NCCL)
    except RuntimeError as e:
        if "unavailable" in str(e):                  # libnccl.so.2 not loadable in this process
            pytest.skip(f"NCCL transport unavailable: {e}")
        raise
    info = rt.rt_dist_info(R.ctx)
    assert info["world"] == 1 and info["transport"] == "nccl"
    streams = [torch.cuda.Stream() for _ in range(3)]
    fbs = []
    for k in range(N_FRAMES):
        fmt = rt.RT_FORMAT_RGBA8 if k % 4 else rt.RT_FORMAT_RGBA16F
        fb = R.alloc_fb(s.width, s.height, fmt)
        fb.zero_()
        streams[k % 3].wait_stream(torch.cuda.current_stream())
        fbs.append((fb, fmt))
        R.set_camera(rigs[k % len(rigs)])
        R.render(s.width, s.height, s.max_depth, fmt=fmt, fb=fb, stream=streams[k % 3])
    torch.cuda.synchronize()
    assert rt.rt_dist_info(R.ctx)["frames"] == N_FRAMES
    rt.rt_dist_finalize(R.ctx)
    bad = []
    for k, (fb, fmt) in enumerate(fbs):
        R.set_camera(rigs[k % len(rigs)])
        ref = R.render(s.width, s.height, s.max_depth, fmt=fmt)["fb"]
        torch.cuda.synchronize()
        if not torch.equal(fb, ref):
            bad.append(k)
    R.close()
    assert not bad, bad
