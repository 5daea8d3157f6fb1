"""Frames in flight (rt_render_stereo_async / rt_download_after): renders enqueued on several
streams of one context run concurrently on the device, each with its own work queue; every
frame must equal the same frame rendered alone, bit for bit, and downloads ordered after a
frame's stream must see the finished frame."""
import ctypes
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1702_01530_b200 import rt, scenes  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = rt.StereoRenderer(0)
    yield r
    r.close()


def test_frames_in_flight_bit_exact(R):
    s = scenes.scene_c3().with_view(width=200, height=120)
    R.upload(s)
    rigs = [scenes.c5_rig(k) for k in range(6)]          # a different camera per frame
    ref = []
    for rg in rigs:
        R.set_camera(rg)
        ref.append(R.render(s.width, s.height, s.max_depth, want_id=True)["fb"])
    torch.cuda.synchronize()
    ref = [x.clone() for x in ref]
    streams = [torch.cuda.Stream() for _ in range(3)]
    fbs = [R.alloc_fb(s.width, s.height) for _ in range(len(rigs))]
    for f in fbs:
        f.zero_()
    torch.cuda.synchronize()
    for k, rg in enumerate(rigs):                         # camera read at enqueue time
        R.set_camera(rg)
        R.render(s.width, s.height, s.max_depth, fb=fbs[k], stream=streams[k % 3])
    torch.cuda.synchronize()
    for k in range(len(rigs)):
        assert torch.equal(fbs[k], ref[k]), f"frame {k} differs when rendered in flight"


def test_sharded_frames_in_flight_cover_the_image(R):
    """Tile shards of one frame rendered concurrently on different streams (the per-GPU launches
    of an N-GPU run, here all on one device) assemble to the single-launch image."""
    s = scenes.scene_c2().with_view(width=150, height=90, max_depth=3)
    R.upload(s)
    R.set_camera(s.rig)
    ref = R.render(s.width, s.height, s.max_depth)["fb"].clone()
    for world in (2, 3, 8):
        fb = R.alloc_fb(s.width, s.height)
        fb.zero_()
        streams = [torch.cuda.Stream() for _ in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            R.render(s.width, s.height, s.max_depth, fb=fb, shard=(r, world), stream=streams[r])
        torch.cuda.synchronize()
        assert torch.equal(fb, ref), f"world {world}"


def test_download_after_stream(R):
    s = scenes.scene_c1()
    R.upload(s)
    R.set_camera(s.rig)
    st = torch.cuda.Stream()
    fb = R.alloc_fb(s.width, s.height)
    n = fb.numel()
    host = rt.rt_host_alloc(n)
    try:
        R.render(s.width, s.height, s.max_depth, fb=fb, stream=st)
        ev = rt.rt_download_after(R.ctx, fb.data_ptr(), host, n, st.cuda_stream)
        rt.rt_wait(ev)
        got = np.frombuffer((ctypes.c_uint8 * n).from_address(host), np.uint8).copy()
        torch.cuda.synchronize()
        assert np.array_equal(got, fb.cpu().numpy().reshape(-1))
    finally:
        rt.rt_host_free(host)


def test_more_renders_in_flight_than_work_queues(R):
    """40 renders on 3 streams with no host synchronisation between them: more than the
    library's 16 work-queue slots, so slots are reused while an earlier render on another stream
    may still drain its queue.  The reuse waits for that render on the device (per-slot
    completion events), so every frame equals the same frame rendered alone."""
    s = scenes.scene_c2().with_view(width=96, height=64, max_depth=3)
    R.upload(s)
    rigs = [scenes.c5_rig(k) for k in range(5)]
    ref = []
    for rg in rigs:
        R.set_camera(rg)
        ref.append(R.render(s.width, s.height, s.max_depth)["fb"].clone())
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(3)]
    fbs = [R.alloc_fb(s.width, s.height) for _ in range(40)]
    for f in fbs:
        f.zero_()
    torch.cuda.synchronize()
    for k in range(40):
        R.set_camera(rigs[k % len(rigs)])
        R.render(s.width, s.height, s.max_depth, fb=fbs[k], stream=streams[k % 3])
    torch.cuda.synchronize()
    for k in range(40):
        assert torch.equal(fbs[k], ref[k % len(rigs)]), f"render {k} (slot {k % 16}) differs"


def test_scene_change_waits_for_renders_in_flight(R):
    """rt_scene_upload / rt_scene_update_vertices free or rewrite buffers that renders still in
    flight on other streams read: they wait for those renders first, so frames enqueued before
    the change show the old scene, bit for bit."""
    a = scenes.scene_c3().with_view(width=160, height=96)
    b = scenes.paper_scene(5).with_view(width=160, height=96)
    R.upload(a)
    R.set_camera(a.rig)
    ref_a = R.render(a.width, a.height, a.max_depth)["fb"].clone()
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(4)]
    fbs = [R.alloc_fb(a.width, a.height) for _ in range(8)]
    torch.cuda.synchronize()
    for k in range(8):
        R.render(a.width, a.height, a.max_depth, fb=fbs[k], stream=streams[k % 4])
    R.upload(b)                                   # no host sync before the new scene replaces a
    torch.cuda.synchronize()
    for k in range(8):
        assert torch.equal(fbs[k], ref_a), f"frame {k} saw the replaced scene"
    # refit while renders are in flight: the earlier frames keep the unmoved geometry
    R.upload(a)
    R.set_camera(a.rig)
    torch.cuda.synchronize()
    for k in range(8):
        R.render(a.width, a.height, a.max_depth, fb=fbs[k], stream=streams[k % 4])
    rt.rt_scene_update_vertices(R.ctx, a.vertices * 1.05)
    torch.cuda.synchronize()
    for k in range(8):
        assert torch.equal(fbs[k], ref_a), f"frame {k} saw the refit"


_BLOCK_CODE = r"""
import sys; sys.path.insert(0, %r)
import numpy as np, torch
from paper_1702_01530_b200 import rt, scenes
R = rt.StereoRenderer(0)
s = scenes.scene_c2().with_view(width=93, height=61, max_depth=3)
R.upload(s); R.set_camera(s.rig)
ref = R.render(s.width, s.height, s.max_depth)["fb"].clone()
for world in (3, 4, 8):
    fb = R.alloc_fb(s.width, s.height); fb.zero_()
    per = rt.rt_shard_bytes(s.width, s.height, world)
    gathered = torch.zeros(world * per, dtype=torch.uint8, device="cuda")
    for r in range(world):
        R.render(s.width, s.height, s.max_depth, fb=fb, shard=(r, world))
        R.render(s.width, s.height, s.max_depth, fb=False, shard=(r, world), shard_buf=gathered[r * per:(r + 1) * per])
    fb2 = torch.zeros_like(fb)
    rt.rt_unpack_shards(R.ctx, gathered.data_ptr(), s.width, s.height, world, rt.RT_FORMAT_RGBA8,
                        rt.rt_fb(fb2[0].data_ptr(), 0, s.width * 4), rt.rt_fb(fb2[1].data_ptr(), 0, s.width * 4))
    torch.cuda.synchronize()
    assert torch.equal(fb, ref), world
    assert torch.equal(fb2, ref), world
print("ok")
"""


def test_block_shard_layout_bit_exact():
    """RT_SHARD_BLOCK=4 (tile pairs dealt in 4x4-tile blocks): every rank's shard
    rendered into the frame, and packed + unpacked on the device, gives the single-launch image."""
    import subprocess
    env = dict(os.environ, RT_SHARD_BLOCK="4")
    r = subprocess.run([sys.executable, "-c", _BLOCK_CODE % ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
