"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/rt_b200.h
declares, and its pure host logic (shard map, host unpack) is correct.  No GPU needed."""
import os
import re

import numpy as np
import pytest

from paper_1702_01530_b200 import rt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAIRS_AT_2 = os.environ.get("RT_SHARD_PAIRS", "0") not in ("", "0")   # library knob, read once


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rt_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:rt_status|int|const char\*)\s+(rt_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    assert sorted(rt.EXPORTED) == syms
    L = rt.lib()
    for name in syms:
        assert getattr(L, name) is not None
    assert rt.rt_version() == 2


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS only (no PTX / other-arch fallback)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rt.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, out.stdout
    ptx = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-ptx", rt.LIB_PATH], capture_output=True, text=True)
    assert ".ptx" not in ptx.stdout


def test_create_without_device_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a device")
    with pytest.raises(rt.RtError):
        rt.rt_create(0)
    assert rt.rt_last_error() != ""


def test_null_arguments_are_rejected_without_a_device():
    """Every entry point validates its pointers before touching CUDA (error behaviour documented
    in include/rt_b200.h): NULL context / outputs -> RT_ERR_INVALID_ARG."""
    import ctypes as C
    L = rt.lib()
    p = rt.rt_render_params(64, 48, 1, 0, 1, 0)
    o = rt.rt_outputs()
    assert L.rt_render_stereo_ex(None, C.byref(p), C.byref(o)) == rt.RT_ERR_INVALID_ARG
    assert L.rt_render_stereo_async(None, C.byref(p), C.byref(o), None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_download_after(None, None, None, 0, None, None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_download(None, None, None, 0, None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_kdtree_build(None, 1, 0, None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_ipc_open(None, None, None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_ipc_close(None, None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_scene_info(None, None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_bench_ceilings(None, None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_intersect(None, None, None, None, 1, 0, None, None, None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_dist_unique_id(None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_dist_init(None, 0, 1, None, 0) == rt.RT_ERR_INVALID_ARG
    assert L.rt_dist_finalize(None) == rt.RT_ERR_INVALID_ARG
    assert L.rt_dist_info(None, None) == rt.RT_ERR_INVALID_ARG
    job = rt.rt_dist_unique_id()
    assert len(job) == rt.RT_DIST_ID_BYTES and any(job) and job != rt.rt_dist_unique_id()
    import ctypes as C2
    h = C2.c_uint64()
    b = (C2.c_char * 128).from_buffer_copy(job)
    assert L.rt_dist_host_selftest(2, 2, C2.cast(b, C2.c_void_p), 1, C2.byref(h)) == rt.RT_ERR_INVALID_ARG   # rank >= world
    assert "NULL" in rt.rt_last_error() or rt.rt_last_error() != ""


@pytest.mark.parametrize("W,H", [(64, 48), (67, 45), (1920, 1080), (17, 1), (1, 1), (33, 200)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
def test_shard_map_exact_cover(W, H, world):
    """PAPER.md:48 'dividing the picture to N identical parts': every tile of both eyes is
    owned by exactly one rank; world 2 is the level-1 eye split."""
    tx, ty = -(-W // 16), -(-H // 16)
    T = tx * ty
    owners = np.full(2 * T, -1)
    counts = []
    for r in range(world):
        ids = rt.rt_shard_tiles(W, H, r, world)
        assert np.all(np.diff(ids.astype(np.int64)) > 0)
        assert np.all(owners[ids] == -1)
        owners[ids] = r
        counts.append(len(ids))
    assert np.all(owners >= 0)
    # tiles are dealt in eye pairs: ranks differ by at most one tile pair
    eye_split = world == 2 and not PAIRS_AT_2
    assert max(counts) - min(counts) <= (1 if eye_split else 2) or T < world
    if eye_split:                                   # G = 2*tile + eye
        assert np.all(owners[0::2] == 0) and np.all(owners[1::2] == 1)
    per = rt.rt_shard_bytes(W, H, world)
    assert per == max(counts) * 256 * 4
    assert rt.rt_shard_bytes(W, H, world, rt.RT_FORMAT_RGBA16F) == 2 * per


def synth_shards(W, H, world):
    """Each rank fills its packed shard with a code of (eye, px, py) using only the shard map."""
    per = rt.rt_shard_bytes(W, H, world) // 4
    tx = -(-W // 16)
    T = tx * -(-H // 16)
    buf = np.zeros((world, per), np.uint32)
    for r in range(world):
        for lt, g in enumerate(rt.rt_shard_tiles(W, H, r, world)):
            eye, t = int(g) & 1, int(g) >> 1
            w = np.arange(256)
            px = (t % tx) * 16 + w % 16
            py = (t // tx) * 16 + w // 16
            buf[r, lt * 256:(lt + 1) * 256] = (eye << 30) | (py << 15) | px
    return buf


def expected_image(W, H):
    py, px = np.mgrid[0:H, 0:W]
    return np.stack([(e << 30) | (py << 15) | px for e in (0, 1)]).astype(np.uint32)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_host_unpack_roundtrip(world):
    W, H = 93, 61
    g = synth_shards(W, H, world)
    L, R = rt.rt_unpack_shards_host(g.view(np.uint8).reshape(-1), W, H, world)
    got = np.stack([L, R]).view(np.uint32)[..., 0]
    np.testing.assert_array_equal(got, expected_image(W, H))


def test_shard_pairs_knob_at_world_2():
    """RT_SHARD_PAIRS=1 deals tile pairs round-robin at world 2 too: both eyes of a
    tile on one rank, exact cover, and the host unpack still reassembles the image."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from paper_1702_01530_b200 import rt\n"
        "import test_abi as t\n"
        "W, H = 93, 61; T = 6 * 4\n"
        "a, b = (rt.rt_shard_tiles(W, H, r, 2).astype(int) for r in (0, 1))\n"
        "assert sorted(np.concatenate([a, b]).tolist()) == list(range(2 * T))\n"
        "assert set(a >> 1).isdisjoint(set(b >> 1))\n"
        "assert len(a) == len(b) and all(((g >> 1) == (h >> 1)) for g, h in zip(a[0::2], a[1::2]))\n"
        "g = t.synth_shards(W, H, 2)\n"
        "L, R = rt.rt_unpack_shards_host(g.view(np.uint8).reshape(-1), W, H, 2)\n"
        "np.testing.assert_array_equal(np.stack([L, R]).view(np.uint32)[..., 0], t.expected_image(W, H))\n"
        "print('ok')\n") % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, RT_SHARD_PAIRS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr


@pytest.mark.parametrize("block", [2, 3, 8])
def test_shard_block_layout(block):
    """RT_SHARD_BLOCK=B: tile pairs dealt to ranks in B x B blocks of tiles -- exact
    cover of both eyes, both eyes of a tile on one rank, every rank's tiles grouped by block, and
    the host unpack reassembles the image for worlds 3, 4 and 8."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from paper_1702_01530_b200 import rt\n"
        "import test_abi as t\n"
        "B = %d\n"
        "for W, H in ((93, 61), (1920, 1080), (17, 40)):\n"
        "    tx, ty = -(-W // 16), -(-H // 16); T = tx * ty\n"
        "    for world in (3, 4, 8):\n"
        "        ids = [rt.rt_shard_tiles(W, H, r, world).astype(int) for r in range(world)]\n"
        "        allg = np.concatenate(ids)\n"
        "        assert sorted(allg.tolist()) == list(range(2 * T)), (W, H, world)\n"
        "        for r, a in enumerate(ids):\n"
        "            assert all(((g >> 1) == (h >> 1)) and g %% 2 == 0 and h == g + 1 for g, h in zip(a[0::2], a[1::2]))\n"
        "            blocks = [((g >> 1) %% tx // B) + (((g >> 1) // tx) // B) * (-(-tx // B)) for g in a[0::2]]\n"
        "            assert all(b %% world == r for b in blocks) and blocks == sorted(blocks)\n"
        "        g = t.synth_shards(W, H, world)\n"
        "        L, R = rt.rt_unpack_shards_host(g.view(np.uint8).reshape(-1), W, H, world)\n"
        "        np.testing.assert_array_equal(np.stack([L, R]).view(np.uint32)[..., 0], t.expected_image(W, H))\n"
        "print('ok')\n") % (ROOT, os.path.join(ROOT, "tests"), block)
    env = dict(os.environ, RT_SHARD_BLOCK=str(block))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_product_package_never_touches_the_oracle():
    """The product path must not import/link/execute oracle/ (it is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_1702_01530_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")) or f == "Makefile":
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|whitted_oracle|oracle\.py)", txt), \
                    os.path.join(dirpath, f)
