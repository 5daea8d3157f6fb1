"""ctypes front-end of the CPU oracle (whitted_oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  The product package never does.

It marshals a `scenes.Scene` into the oracle's C structs; every piece of
ray-tracing arithmetic lives in whitted_oracle.c (double precision, brute force).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

FRAG_COMPETE, FRAG_BOUNDARY, FRAG_GRAZE, FRAG_RANGE, FRAG_SHADE, FRAG_SHADOW, FRAG_UNSTABLE = 1, 2, 4, 8, 16, 32, 64
ID_FRAGILE_MASK = FRAG_COMPETE | FRAG_BOUNDARY | FRAG_GRAZE | FRAG_RANGE


class OracleScene(C.Structure):
    _fields_ = [
        ("n_spheres", C.c_int32), ("spheres", C.POINTER(C.c_double)), ("sphere_mat", C.POINTER(C.c_int32)),
        ("n_planes", C.c_int32), ("planes", C.POINTER(C.c_double)), ("plane_mat", C.POINTER(C.c_int32)),
        ("n_vertices", C.c_int32), ("vertices", C.POINTER(C.c_double)),
        ("n_tris", C.c_int32), ("tris", C.POINTER(C.c_int32)), ("tri_mat", C.POINTER(C.c_int32)),
        ("n_mats", C.c_int32), ("mats", C.POINTER(C.c_double)),
        ("n_lights", C.c_int32), ("lights", C.POINTER(C.c_double)),
        ("ambient", C.c_double * 3), ("background", C.c_double * 3),
    ]


class OracleCam(C.Structure):
    _fields_ = [
        ("eye", (C.c_double * 3) * 2), ("f", C.c_double * 3), ("r", C.c_double * 3), ("u", C.c_double * 3),
        ("th", C.c_double), ("aspect", C.c_double), ("sigma", C.c_double * 2),
        ("width", C.c_int32), ("height", C.c_int32),
    ]


class OracleEps(C.Structure):
    _fields_ = [("eps_t", C.c_double), ("eps_sphere", C.c_double), ("eps_edge", C.c_double),
                ("eps_abs", C.c_double), ("perturb", C.c_double), ("perturb_tol", C.c_double)]


CAND_K = 8          # near-tie candidate IDs kept per ID-fragile pixel

# eps_edge 1e-6: SURVEY §8(c) #22 sets the triangle-edge band to >= 4x the largest edge margin of
# any GPU/oracle ID disagreement; the round-2 reports (profiles/r02_parity_report_eps1e-*.json:
# 0.52 M C3 pixels, C4 and C5 samples) saw no disagreement at all, off or on the band, and the
# FP32 edge-decision error is ~1e-7 angular (reading 22).
DEFAULT_EPS = dict(eps_t=1e-4, eps_sphere=1e-4, eps_edge=1e-6, eps_abs=1e-5, perturb=1e-6, perturb_tol=1e-3)

_lib = None


def build(force=False):
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "whitted_oracle.c")):
        subprocess.run(["make", "-s", "-C", _HERE, "CC=gcc"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        L.oracle_setup_rig.argtypes = [dp, dp, dp, C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int32,
                                       C.POINTER(OracleCam)]
        L.oracle_setup_rig.restype = C.c_int
        L.oracle_primary_ray.argtypes = [C.POINTER(OracleCam), C.c_int32, C.c_int32, C.c_int32, dp, dp]
        L.oracle_primary_ray.restype = None
        L.oracle_nearest.argtypes = [C.POINTER(OracleScene), dp, dp, dp, C.POINTER(C.c_int32)]
        L.oracle_nearest.restype = C.c_int
        L.oracle_trace_ray.argtypes = [C.POINTER(OracleScene), dp, dp, C.c_int32, dp, C.POINTER(C.c_longlong)]
        L.oracle_trace_ray.restype = None
        L.oracle_half_bits.argtypes = [C.c_double]
        L.oracle_half_bits.restype = C.c_uint16
        L.oracle_render.argtypes = [C.POINTER(OracleScene), C.POINTER(OracleCam), C.c_int32, C.c_int64,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(OracleEps), C.c_int32,
                                    C.c_void_p, C.c_int32, C.c_void_p]
        L.oracle_render.restype = C.c_int
        L.oracle_trace_ray_ex.argtypes = [C.POINTER(OracleScene), dp, dp, C.c_int32, C.POINTER(OracleEps), dp,
                                          C.POINTER(C.c_longlong), C.POINTER(C.c_uint32)]
        L.oracle_trace_ray_ex.restype = None
        L.oracle_ray_flags.argtypes = [C.POINTER(OracleScene), dp, dp, C.c_int32, C.c_double, C.POINTER(OracleEps), dp]
        L.oracle_ray_flags.restype = C.c_uint32
        L.oracle_ray_candidates.argtypes = [C.POINTER(OracleScene), dp, dp, C.POINTER(OracleEps), C.c_void_p,
                                            C.c_int32]
        L.oracle_ray_candidates.restype = C.c_int32
        L.oracle_version.restype = C.c_int
        for fn in (L.oracle_compose_anaglyph, L.oracle_compose_sbs):
            fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
            fn.restype = None
        _lib = L
    return _lib


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class Oracle:
    """Holds the C-side view of one scene (keeps the numpy buffers alive)."""

    def __init__(self, scene):
        self.scene = scene
        L = lib()
        self._keep = []

        def d(a, shape_last):
            a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, shape_last) if shape_last else
                                     np.asarray(a, np.float64))
            self._keep.append(a)
            return a

        def i(a):
            a = np.ascontiguousarray(np.asarray(a, np.int64).astype(np.int32).reshape(-1))
            self._keep.append(a)
            return a

        sp, pl, vt = d(scene.spheres, 4), d(scene.planes, 4), d(scene.vertices, 3)
        ma, li = d(scene.materials, 10), d(scene.lights, 6)
        spm, plm, tr, trm = i(scene.sphere_mat), i(scene.plane_mat), i(scene.tris), i(scene.tri_mat)
        st = OracleScene()
        st.n_spheres, st.spheres, st.sphere_mat = len(sp), _dptr(sp), _iptr(spm)
        st.n_planes, st.planes, st.plane_mat = len(pl), _dptr(pl), _iptr(plm)
        st.n_vertices, st.vertices = len(vt), _dptr(vt)
        st.n_tris, st.tris, st.tri_mat = len(trm), _iptr(tr), _iptr(trm)
        st.n_mats, st.mats = len(ma), _dptr(ma)
        st.n_lights, st.lights = len(li), _dptr(li)
        for k in range(3):
            st.ambient[k] = float(scene.ambient[k])
            st.background[k] = float(scene.background[k])
        self.st = st
        self.L = L

    # ---- camera
    def camera(self, rig=None, width=None, height=None):
        rig = rig or self.scene.rig
        width = width or self.scene.width
        height = height or self.scene.height
        cam = OracleCam()
        e = np.ascontiguousarray(rig.eye, np.float64)
        la = np.ascontiguousarray(rig.look_at, np.float64)
        up = np.ascontiguousarray(rig.up, np.float64)
        rc = self.L.oracle_setup_rig(_dptr(e), _dptr(la), _dptr(up), rig.vfov_deg, rig.interocular,
                                     rig.convergence, width, height, C.byref(cam))
        if rc != 0:
            raise ValueError("invalid camera")
        return cam

    def primary_ray(self, cam, eye, px, py):
        o = np.zeros(3)
        dd = np.zeros(3)
        self.L.oracle_primary_ray(C.byref(cam), eye, px, py, _dptr(o), _dptr(dd))
        return o, dd

    def nearest(self, o, d):
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        t = C.c_double()
        pid = C.c_int32()
        self.L.oracle_nearest(C.byref(self.st), _dptr(o), _dptr(d), C.byref(t), C.byref(pid))
        return t.value, pid.value

    def trace_ray(self, o, d, depth):
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        rgb = np.zeros(3)
        cnt = (C.c_longlong * 4)()
        self.L.oracle_trace_ray(C.byref(self.st), _dptr(o), _dptr(d), depth, _dptr(rgb), cnt)
        return rgb, np.array(list(cnt), np.int64)

    @staticmethod
    def _eps(eps):
        return OracleEps(**{**DEFAULT_EPS, **(eps or {})})

    def trace_ray_ex(self, o, d, depth, eps=None):
        """One ray with the fragility analysis: (unclamped rgb, counts, tree flags)."""
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        rgb = np.zeros(3)
        cnt = (C.c_longlong * 4)()
        fl = C.c_uint32()
        e = self._eps(eps)
        self.L.oracle_trace_ray_ex(C.byref(self.st), _dptr(o), _dptr(d), depth, C.byref(e), _dptr(rgb), cnt,
                                   C.byref(fl))
        return rgb, np.array(list(cnt), np.int64), fl.value

    def ray_flags(self, o, d, kind="nearest", dist=0.0, eps=None):
        """Fragility flags of one nearest (F1-F5) or shadow (over (t_min, dist)) query -> (flags, margin)."""
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        mg = C.c_double(0.0)
        e = self._eps(eps)
        f = self.L.oracle_ray_flags(C.byref(self.st), _dptr(o), _dptr(d), 0 if kind == "nearest" else 1, float(dist),
                                    C.byref(e), C.byref(mg))
        return int(f), mg.value

    def ray_candidates(self, o, d, eps=None, kmax=CAND_K):
        """Near-tie candidate IDs of the nearest query along (o, d) (-1 = miss) -> (sorted list, count)."""
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        buf = np.full(kmax, -2, np.int32)
        e = self._eps(eps)
        n = self.L.oracle_ray_candidates(C.byref(self.st), _dptr(o), _dptr(d), C.byref(e), buf.ctypes.data, kmax)
        return sorted(int(x) for x in buf[:min(n, kmax)]), int(n)

    def render(self, rig=None, width=None, height=None, max_depth=None, pixels=None, eps=None,
               flags=True, threads=0):
        """Render both eyes (pixels=None) or a list of (eye, px, py) triples.

        Returns a dict of numpy arrays: radiance (n,3) unclamped, rgba8 (n,4) u8,
        rgba16 (n,4) u16 binary16 bits, id (n,), pflags, tflags, margin, counts (4,).
        Full renders are reshaped to (2, H, W, ...).
        """
        width = width or self.scene.width
        height = height or self.scene.height
        max_depth = self.scene.max_depth if max_depth is None else max_depth
        cam = self.camera(rig, width, height)
        if pixels is None:
            n = 2 * width * height
            pix = None
        else:
            pix = np.ascontiguousarray(np.asarray(pixels, np.int32).reshape(-1, 3))
            n = len(pix)
        rad = np.zeros((n, 3))
        q8 = np.zeros((n, 4), np.uint8)
        h16 = np.zeros((n, 4), np.uint16)
        ids = np.zeros(n, np.int32)
        pf = np.zeros(n, np.uint32)
        tf = np.zeros(n, np.uint32)
        mg = np.zeros(n)
        cnt = np.zeros(4, np.int64)
        cand = np.full((n, CAND_K), -2, np.int32)
        ncand = np.zeros(n, np.int32)
        e = None
        if flags:
            e = self._eps(eps)
        rc = self.L.oracle_render(C.byref(self.st), C.byref(cam), max_depth, n,
                                  None if pix is None else pix.ctypes.data,
                                  rad.ctypes.data, q8.ctypes.data, h16.ctypes.data, ids.ctypes.data,
                                  pf.ctypes.data, tf.ctypes.data, mg.ctypes.data, cnt.ctypes.data,
                                  None if e is None else C.byref(e), int(threads),
                                  cand.ctypes.data if flags else None, CAND_K, ncand.ctypes.data if flags else None)
        if rc != 0:
            raise ValueError("oracle_render failed")
        out = dict(radiance=rad, rgba8=q8, rgba16=h16, id=ids, pflags=pf, tflags=tf, margin=mg, counts=cnt,
                   cand=cand, ncand=ncand)
        if pixels is None:
            for k in ("radiance", "rgba8", "rgba16", "cand"):
                out[k] = out[k].reshape(2, height, width, -1)
            for k in ("id", "pflags", "tflags", "margin", "ncand"):
                out[k] = out[k].reshape(2, height, width)
        return out


def half_bits(x):
    return lib().oracle_half_bits(float(x))


def compose(left, right, mode):
    """SPEC compose_anaglyph / compose_sbs on (H, W, 4) uint8 arrays; mode 'anaglyph' | 'sbs'."""
    L = np.ascontiguousarray(left, np.uint8)
    R = np.ascontiguousarray(right, np.uint8)
    H, W = L.shape[:2]
    if mode == "anaglyph":
        out = np.zeros((H, W, 4), np.uint8)
        lib().oracle_compose_anaglyph(L.ctypes.data, R.ctypes.data, W, H, out.ctypes.data)
    else:
        out = np.zeros((H, 2 * (W // 2), 4), np.uint8)
        lib().oracle_compose_sbs(L.ctypes.data, R.ctypes.data, W, H, out.ctypes.data)
    return out
