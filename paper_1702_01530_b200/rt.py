"""Thin Python binding of the C ABI in include/rt_b200.h (argument marshalling only).

Every function named rt_* here calls the C entry point of the same name in the in-tree
library paper_1702_01530_b200/lib/librt_b200.so; all ray tracing runs in its CUDA kernels.
There is no CPU fallback: if the library is missing this module raises on import-time use.
PyTorch is used only for device memory, streams and (in bench.py) process groups.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RT_LIB_PATH") or os.path.join(_HERE, "lib", "librt_b200.so")   # override: experiments only

RT_OK, RT_ERR_INVALID_ARG, RT_ERR_CUDA, RT_ERR_OOM, RT_ERR_NO_SCENE, RT_ERR_NO_CAMERA, RT_ERR_SIZE, \
    RT_ERR_NOT_READY, RT_ERR_PEER = range(9)
RT_FORMAT_RGBA8, RT_FORMAT_RGBA16F = 0, 1
RT_RENDER_COUNT, RT_RENDER_BRUTE_FORCE, RT_RENDER_PEER_STORE, RT_RENDER_KDTREE = 1, 2, 4, 8
RT_NUM_COUNTERS = 13
RT_COMPOSE_ANAGLYPH, RT_COMPOSE_SBS = 0, 1
RT_TILE = 16
RT_DIST_ID_BYTES = 128
RT_DIST_PEER, RT_DIST_NCCL = 0, 1
COUNTER_NAMES = ["primary", "reflection", "refraction", "shadow", "node_visits", "tri_tests", "sphere_tests",
                 "plane_tests", "shade_hits", "light_evals", "misses", "pixels", "box_tests"]

# Every symbol include/rt_b200.h declares (checked by tests/test_abi.py).
EXPORTED = ["rt_create", "rt_destroy", "rt_synchronize", "rt_last_error", "rt_version", "rt_scene_upload",
            "rt_set_stereo_camera", "rt_render_stereo", "rt_render_stereo_ex", "rt_download", "rt_wait", "rt_query",
            "rt_host_alloc", "rt_host_free", "rt_upload", "rt_shard_tiles", "rt_shard_bytes", "rt_unpack_shards_host",
            "rt_unpack_shards", "rt_ipc_get_handle", "rt_ipc_open", "rt_ipc_close", "rt_scene_info", "rt_bvh_export",
            "rt_bench_ffma", "rt_compose", "rt_scene_update_vertices", "rt_bvh_width", "rt_kdtree_build",
            "rt_render_stereo_async", "rt_download_after", "rt_bench_ceilings", "rt_dist_unique_id", "rt_dist_init",
            "rt_dist_finalize", "rt_dist_info", "rt_dist_host_selftest", "rt_intersect"]


class RtError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"rt status {status}: {msg}")
        self.status = status


class rt_primitives(C.Structure):
    _fields_ = [("spheres", C.c_void_p), ("sphere_mat", C.c_void_p), ("n_spheres", C.c_uint32),
                ("planes", C.c_void_p), ("plane_mat", C.c_void_p), ("n_planes", C.c_uint32),
                ("vertices", C.c_void_p), ("n_vertices", C.c_uint32),
                ("tri_indices", C.c_void_p), ("tri_mat", C.c_void_p), ("n_triangles", C.c_uint32)]


class rt_material(C.Structure):
    _fields_ = [("kd", C.c_float * 3), ("ks", C.c_float * 3), ("shininess", C.c_float), ("kr", C.c_float),
                ("kt", C.c_float), ("ior", C.c_float)]


class rt_light(C.Structure):
    _fields_ = [("pos", C.c_float * 3), ("intensity", C.c_float * 3)]


class rt_env(C.Structure):
    _fields_ = [("ambient", C.c_float * 3), ("background", C.c_float * 3)]


class rt_fb(C.Structure):
    _fields_ = [("dev_ptr", C.c_void_p), ("format", C.c_uint32), ("pitch_bytes", C.c_uint64)]


class rt_render_params(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("max_depth", C.c_uint32),
                ("shard_rank", C.c_uint32), ("shard_world", C.c_uint32), ("flags", C.c_uint32)]


class rt_outputs(C.Structure):
    _fields_ = [("left", rt_fb), ("right", rt_fb), ("prim_id", C.c_void_p), ("radiance", C.c_void_p),
                ("shard", C.c_void_p), ("shard_format", C.c_uint32), ("counters", C.c_void_p),
                ("composed", rt_fb), ("compose_mode", C.c_uint32)]


_lib = None


def lib():
    """Load the in-tree CUDA library; fail loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, f32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_float
        sig = {
            "rt_create": [C.c_int, vp, C.POINTER(vp)],
            "rt_destroy": [vp], "rt_synchronize": [vp],
            "rt_scene_upload": [vp, C.POINTER(rt_primitives), vp, u32, vp, u32, C.POINTER(rt_env)],
            "rt_set_stereo_camera": [vp, vp, vp, vp, f32, f32, f32],
            "rt_render_stereo": [vp, u32, u32, u32, rt_fb, rt_fb],
            "rt_render_stereo_ex": [vp, C.POINTER(rt_render_params), C.POINTER(rt_outputs)],
            "rt_download": [vp, vp, vp, C.c_size_t, C.POINTER(vp)],
            "rt_render_stereo_async": [vp, C.POINTER(rt_render_params), C.POINTER(rt_outputs), vp],
            "rt_download_after": [vp, vp, vp, C.c_size_t, vp, C.POINTER(vp)],
            "rt_wait": [vp], "rt_query": [vp],
            "rt_host_alloc": [C.c_size_t, C.POINTER(vp)], "rt_host_free": [vp],
            "rt_upload": [vp, vp, vp, C.c_size_t],
            "rt_shard_tiles": [u32, u32, u32, u32, C.POINTER(u32), vp],
            "rt_shard_bytes": [u32, u32, u32, u32, C.POINTER(u64)],
            "rt_unpack_shards_host": [vp, u32, u32, u32, u32, vp, vp, u64],
            "rt_unpack_shards": [vp, vp, u32, u32, u32, u32, rt_fb, rt_fb],
            "rt_ipc_get_handle": [vp, vp, C.POINTER(u64)], "rt_ipc_open": [vp, vp, C.POINTER(vp)], "rt_ipc_close": [vp, vp],
            "rt_scene_info": [vp, vp],
            "rt_bvh_export": [vp, vp, C.POINTER(u32), vp, C.POINTER(u32)],
            "rt_intersect": [vp, vp, vp, vp, u32, u32, vp, vp, vp],
            "rt_bench_ffma": [vp, u32, C.POINTER(C.c_double), C.POINTER(C.c_double)],
            "rt_compose": [vp, rt_fb, rt_fb, u32, u32, u32, rt_fb],
            "rt_scene_update_vertices": [vp, vp, u32],
            "rt_kdtree_build": [vp, u32, u32, vp],
            "rt_bench_ceilings": [vp, vp],
            "rt_dist_unique_id": [vp], "rt_dist_init": [vp, C.c_int, C.c_int, vp, u32], "rt_dist_finalize": [vp],
            "rt_dist_info": [vp, vp],
            "rt_dist_host_selftest": [C.c_int, C.c_int, vp, u32, C.POINTER(u64)],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.rt_last_error.restype = C.c_char_p
        L.rt_last_error.argtypes = []
        L.rt_version.restype = C.c_int
        L.rt_bvh_width.restype = C.c_int
        _lib = L
    return _lib


def _check(status):
    if status != RT_OK:
        raise RtError(status, lib().rt_last_error().decode(errors="replace"))
    return status


def _ptr(a):
    return None if a is None else a.ctypes.data


def _f3(x):
    return (C.c_float * 3)(*[float(v) for v in np.asarray(x, np.float64).reshape(3)])


# ---------------------------------------------------------------- raw entry points (same names)
def rt_version():
    return lib().rt_version()


def rt_bvh_width():
    return lib().rt_bvh_width()


def rt_last_error():
    return lib().rt_last_error().decode(errors="replace")


def rt_create(device=0, stream=None):
    out = C.c_void_p()
    _check(lib().rt_create(int(device), stream, C.byref(out)))
    return out.value


def rt_destroy(ctx):
    return _check(lib().rt_destroy(ctx))


def rt_synchronize(ctx):
    return _check(lib().rt_synchronize(ctx))


class SceneArrays:
    """C-side view of a scenes.Scene (float32 / uint32 copies kept alive during the call)."""

    def __init__(self, scene):
        f32 = lambda a, k: np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, k), dtype=np.float32)
        u32 = lambda a: np.ascontiguousarray(np.asarray(a).reshape(-1), dtype=np.uint32)
        self.spheres, self.sphere_mat = f32(scene.spheres, 4), u32(scene.sphere_mat)
        self.planes, self.plane_mat = f32(scene.planes, 4), u32(scene.plane_mat)
        self.vertices = f32(scene.vertices, 3)
        self.tris, self.tri_mat = u32(scene.tris), u32(scene.tri_mat)
        m = np.asarray(scene.materials, np.float64).reshape(-1, 10)
        self.mats = (rt_material * max(1, len(m)))()
        for i, row in enumerate(m):
            self.mats[i] = rt_material((C.c_float * 3)(*row[0:3]), (C.c_float * 3)(*row[3:6]), row[6], row[7],
                                       row[8], row[9])
        self.n_mats = len(m)
        li = np.asarray(scene.lights, np.float64).reshape(-1, 6)
        self.lights = (rt_light * max(1, len(li)))()
        for i, row in enumerate(li):
            self.lights[i] = rt_light((C.c_float * 3)(*row[0:3]), (C.c_float * 3)(*row[3:6]))
        self.n_lights = len(li)
        self.env = rt_env(_f3(scene.ambient), _f3(scene.background))
        self.prims = rt_primitives(_ptr(self.spheres), _ptr(self.sphere_mat), len(self.spheres),
                                   _ptr(self.planes), _ptr(self.plane_mat), len(self.planes),
                                   _ptr(self.vertices), len(self.vertices),
                                   _ptr(self.tris), _ptr(self.tri_mat), len(self.tri_mat))


def rt_scene_upload(ctx, scene):
    a = SceneArrays(scene)
    _check(lib().rt_scene_upload(ctx, C.byref(a.prims), C.cast(a.mats, C.c_void_p), a.n_mats,
                                 C.cast(a.lights, C.c_void_p), a.n_lights, C.byref(a.env)))


def rt_scene_update_vertices(ctx, vertices):
    v = np.ascontiguousarray(np.asarray(vertices, np.float64).reshape(-1, 3), dtype=np.float32)
    _check(lib().rt_scene_update_vertices(ctx, v.ctypes.data, len(v)))


def rt_set_stereo_camera(ctx, eye, look_at, up, vfov_deg, interocular, convergence):
    e, la, u = _f3(eye), _f3(look_at), _f3(up)
    _check(lib().rt_set_stereo_camera(ctx, C.cast(e, C.c_void_p), C.cast(la, C.c_void_p), C.cast(u, C.c_void_p),
                                      float(vfov_deg), float(interocular), float(convergence)))


def make_fb(dev_ptr, fmt=RT_FORMAT_RGBA8, pitch=0):
    return rt_fb(dev_ptr, fmt, pitch)


def rt_render_stereo(ctx, width, height, max_depth, out_left, out_right):
    _check(lib().rt_render_stereo(ctx, width, height, max_depth, out_left, out_right))


def rt_render_stereo_ex(ctx, params, outputs):
    _check(lib().rt_render_stereo_ex(ctx, C.byref(params), C.byref(outputs)))


def rt_render_stereo_async(ctx, params, outputs, cuda_stream):
    _check(lib().rt_render_stereo_async(ctx, C.byref(params), C.byref(outputs), cuda_stream))


def rt_download(ctx, dev_src, host_dst, nbytes, want_event=True):
    ev = C.c_void_p()
    _check(lib().rt_download(ctx, dev_src, host_dst, nbytes, C.byref(ev) if want_event else None))
    return ev.value


def rt_download_after(ctx, dev_src, host_dst, nbytes, after_stream, want_event=True):
    ev = C.c_void_p()
    _check(lib().rt_download_after(ctx, dev_src, host_dst, nbytes, after_stream, C.byref(ev) if want_event else None))
    return ev.value


def rt_upload(ctx, host_src, dev_dst, nbytes):
    _check(lib().rt_upload(ctx, host_src, dev_dst, nbytes))


def rt_wait(ev):
    _check(lib().rt_wait(ev))


def rt_query(ev):
    s = lib().rt_query(ev)
    if s == RT_ERR_NOT_READY:
        return False
    _check(s)
    return True


def rt_host_alloc(nbytes):
    p = C.c_void_p()
    _check(lib().rt_host_alloc(nbytes, C.byref(p)))
    return p.value


def rt_host_free(p):
    _check(lib().rt_host_free(p))


def rt_shard_tiles(width, height, rank, world):
    n = C.c_uint32()
    _check(lib().rt_shard_tiles(width, height, rank, world, C.byref(n), None))
    ids = np.zeros(n.value, np.uint32)
    if n.value:
        _check(lib().rt_shard_tiles(width, height, rank, world, C.byref(n), ids.ctypes.data))
    return ids


def rt_shard_bytes(width, height, world, fmt=RT_FORMAT_RGBA8):
    b = C.c_uint64()
    _check(lib().rt_shard_bytes(width, height, world, fmt, C.byref(b)))
    return b.value


def rt_unpack_shards_host(gathered, width, height, world, fmt=RT_FORMAT_RGBA8):
    """numpy (world*shard_bytes,) u8 -> (left, right) (H, W, 4) u8 or u16 arrays."""
    g = np.ascontiguousarray(gathered).view(np.uint8)
    dt = np.uint8 if fmt == RT_FORMAT_RGBA8 else np.uint16
    left = np.zeros((height, width, 4), dt)
    right = np.zeros((height, width, 4), dt)
    _check(lib().rt_unpack_shards_host(g.ctypes.data, width, height, world, fmt, left.ctypes.data,
                                       right.ctypes.data, left.strides[0]))
    return left, right


def rt_unpack_shards(ctx, gathered_ptr, width, height, world, fmt, left_fb, right_fb):
    _check(lib().rt_unpack_shards(ctx, gathered_ptr, width, height, world, fmt, left_fb, right_fb))


def rt_ipc_get_handle(dev_ptr):
    """-> (64-byte handle of the allocation containing dev_ptr, byte offset of dev_ptr in it)"""
    h = (C.c_char * 64)()
    off = C.c_uint64()
    _check(lib().rt_ipc_get_handle(dev_ptr, C.cast(h, C.c_void_p), C.byref(off)))
    return bytes(h), off.value


def rt_ipc_open(ctx, handle):
    h = (C.c_char * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    _check(lib().rt_ipc_open(ctx, C.cast(h, C.c_void_p), C.byref(p)))
    return p.value


def rt_ipc_close(ctx, dev_ptr):
    _check(lib().rt_ipc_close(ctx, dev_ptr))


def rt_scene_info(ctx):
    a = np.zeros(8, np.uint64)
    _check(lib().rt_scene_info(ctx, a.ctypes.data))
    keys = ["n_spheres", "n_planes", "n_triangles", "bvh_prims", "bvh_nodes", "bvh_depth", "device_bytes", "build_us"]
    return dict(zip(keys, (int(x) for x in a)))


def rt_bvh_export(ctx):
    nn, npr = C.c_uint32(), C.c_uint32()
    _check(lib().rt_bvh_export(ctx, None, C.byref(nn), None, C.byref(npr)))
    nodes = np.zeros((max(nn.value, 1), 7 * lib().rt_bvh_width()), np.float32)
    gids = np.zeros(max(npr.value, 1), np.int32)
    _check(lib().rt_bvh_export(ctx, nodes.ctypes.data, C.byref(nn), gids.ctypes.data, C.byref(npr)))
    return nodes[:nn.value], gids[:npr.value]


RT_QUERY_NEAREST, RT_QUERY_ANY, RT_QUERY_BRUTE_FORCE = 0, 1, 2


def rt_intersect(ctx, o, d, tmax=None, any_hit=False, brute=False, stream=None):
    """Ray queries through the renderer's traversal (rt_b200.h rt_intersect).  o, d: contiguous
    float32 CUDA tensors (n, 3); tmax: (n,) float32 for any-hit queries.  Returns (t, id) CUDA
    tensors for nearest-hit queries, the int32 occlusion flags for any-hit ones (not synchronised)."""
    import torch
    n = o.shape[0]
    ids = torch.empty(n, dtype=torch.int32, device=o.device)
    t = None if any_hit else torch.empty(n, dtype=torch.float32, device=o.device)
    flags = (RT_QUERY_ANY if any_hit else RT_QUERY_NEAREST) | (RT_QUERY_BRUTE_FORCE if brute else 0)
    st = (stream or torch.cuda.current_stream()).cuda_stream
    _check(lib().rt_intersect(ctx, o.data_ptr(), d.data_ptr(), tmax.data_ptr() if tmax is not None else None, n, flags,
                              t.data_ptr() if t is not None else None, ids.data_ptr(), st))
    return ids if any_hit else (t, ids)


def rt_kdtree_build(ctx, max_leaf=1, max_depth=0):
    """NEXT-4 ablation: host-built SAH kd-tree over the uploaded scene (see rt_b200.h)."""
    a = np.zeros(6, np.uint64)
    _check(lib().rt_kdtree_build(ctx, max_leaf, max_depth, a.ctypes.data))
    keys = ["kd_nodes", "kd_refs", "kd_depth", "kd_leaves", "kd_device_bytes", "kd_build_us"]
    return dict(zip(keys, (int(x) for x in a)))


def rt_compose(ctx, left_fb, right_fb, width, height, mode, out_fb):
    _check(lib().rt_compose(ctx, left_fb, right_fb, width, height, mode, out_fb))


def rt_bench_ffma(ctx, iters=2048):
    tf, ms = C.c_double(), C.c_double()
    _check(lib().rt_bench_ffma(ctx, iters, C.byref(tf), C.byref(ms)))
    return tf.value, ms.value


def rt_dist_unique_id():
    """128-byte job id for rt_dist_init (rank 0 creates it, the caller broadcasts it)."""
    b = (C.c_char * RT_DIST_ID_BYTES)()
    _check(lib().rt_dist_unique_id(C.cast(b, C.c_void_p)))
    return bytes(b)


def rt_dist_init(ctx, rank, world, job_id, transport=RT_DIST_PEER):
    b = (C.c_char * RT_DIST_ID_BYTES).from_buffer_copy(job_id)
    _check(lib().rt_dist_init(ctx, int(rank), int(world), C.cast(b, C.c_void_p), int(transport)))


def rt_dist_host_selftest(rank, world, job_id, frames):
    """host half of the multi-GPU protocol, no device work (tests) -> checksum"""
    b = (C.c_char * RT_DIST_ID_BYTES).from_buffer_copy(job_id)
    h = C.c_uint64()
    _check(lib().rt_dist_host_selftest(int(rank), int(world), C.cast(b, C.c_void_p), int(frames), C.byref(h)))
    return h.value


def rt_dist_finalize(ctx):
    _check(lib().rt_dist_finalize(ctx))


def rt_dist_info(ctx):
    a = np.zeros(4, np.int32)
    _check(lib().rt_dist_info(ctx, a.ctypes.data))
    return {"rank": int(a[0]), "world": int(a[1]), "transport": {0: "peer", 1: "nccl"}.get(int(a[2]), "none"),
            "frames": int(a[3])}


CEILING_NAMES = ["ffma_flop_clk_sm", "ffma2_flop_clk_sm", "fmnmx_clk_sm", "fmnmx3_clk_sm", "l1_bytes_clk_sm",
                 "smem_bytes_clk_sm", "sm_mhz"]


def rt_bench_ceilings(ctx):
    """B0 machine ceilings per SM per clock (see rt_b200.h) -> dict"""
    a = np.zeros(len(CEILING_NAMES), np.float64)
    _check(lib().rt_bench_ceilings(ctx, a.ctypes.data))
    return dict(zip(CEILING_NAMES, (float(x) for x in a)))


# ---------------------------------------------------------------- convenience wrapper (torch memory)
class StereoRenderer:
    """One context on one CUDA device, bound to torch's current stream there."""

    def __init__(self, device=0, stream=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        # torch's default stream has handle 0; pass cudaStreamLegacy (0x1) so the library
        # enqueues on that same stream instead of creating its own (NULL) one.
        self.ctx = rt_create(device, stream.cuda_stream or 1)
        self._counters = torch.zeros(RT_NUM_COUNTERS, dtype=torch.int64, device=self.device)
        self.scene = None

    def close(self):
        if self.ctx:
            rt_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, scene):
        rt_scene_upload(self.ctx, scene)
        self.scene = scene
        return rt_scene_info(self.ctx)

    def set_camera(self, rig):
        rt_set_stereo_camera(self.ctx, rig.eye, rig.look_at, rig.up, rig.vfov_deg, rig.interocular, rig.convergence)

    def alloc_fb(self, width, height, fmt=RT_FORMAT_RGBA8):
        t = self.torch
        dt = t.uint8 if fmt == RT_FORMAT_RGBA8 else t.float16
        return t.empty((2, height, width, 4), dtype=dt, device=self.device)

    def render(self, width, height, max_depth, fmt=RT_FORMAT_RGBA8, fb=None, want_id=False, want_radiance=False,
               count=False, brute=False, shard=(0, 1), shard_buf=None, shard_fmt=RT_FORMAT_RGBA8, fb_ptrs=None,
               peer=False, kdtree=False, stream=None, compose=None):
        """Enqueue one stereo render; returns dict of torch device tensors (not synchronised)."""
        t = self.torch
        out = {}
        o = rt_outputs()
        if fb is None and fb_ptrs is None:
            fb = self.alloc_fb(width, height, fmt)
        if fb_ptrs is not None:                     # raw device pointers (e.g. a peer's IPC-mapped FB)
            lp, rp, pitch = fb_ptrs
            o.left = rt_fb(lp, fmt, pitch)
            o.right = rt_fb(rp, fmt, pitch)
        elif fb is not False and fb is not None:
            pitch = fb.stride(1) * fb.element_size()
            o.left = rt_fb(fb[0].data_ptr(), fmt, pitch)
            o.right = rt_fb(fb[1].data_ptr(), fmt, pitch)
            out["fb"] = fb
        if want_id:
            out["id"] = t.full((2, height, width), -2, dtype=t.int32, device=self.device)
            o.prim_id = out["id"].data_ptr()
        if want_radiance:
            out["radiance"] = t.full((2, height, width, 4), float("nan"), dtype=t.float32, device=self.device)
            o.radiance = out["radiance"].data_ptr()
        if compose is not None:                     # (mode, (H, W', 4) u8 tensor): fused composition
            mode, comp = compose
            o.composed = rt_fb(comp.data_ptr(), RT_FORMAT_RGBA8, comp.stride(0) * comp.element_size())
            o.compose_mode = mode
            out["composed"] = comp
        if shard_buf is not None:
            o.shard = shard_buf.data_ptr()
            o.shard_format = shard_fmt
        flags = 0
        if count:
            self._counters.zero_()
            o.counters = self._counters.data_ptr()
            flags |= RT_RENDER_COUNT
        if brute:
            flags |= RT_RENDER_BRUTE_FORCE
        if peer:
            flags |= RT_RENDER_PEER_STORE
        if kdtree:
            flags |= RT_RENDER_KDTREE
        p = rt_render_params(width, height, max_depth, shard[0], shard[1], flags)
        if stream is None:
            rt_render_stereo_ex(self.ctx, p, o)
        else:                                       # a frame in flight on its own torch stream
            stream.wait_stream(t.cuda.current_stream(self.device))   # outputs allocated / filled above
            rt_render_stereo_async(self.ctx, p, o, stream.cuda_stream or 1)
            for v in out.values():                  # keep the caching allocator from reusing them early
                if hasattr(v, "record_stream"):
                    v.record_stream(stream)
            if count:
                self._counters.record_stream(stream)
        if count:
            out["counters"] = self._counters
        return out

    def counters_dict(self, counters):
        v = counters.cpu().numpy()
        return {k: int(x) for k, x in zip(COUNTER_NAMES, v)}
