"""Seeded synthetic scene generators (input fixtures shared by the oracle and the CUDA path).

This module holds NO ray-tracing arithmetic: it only builds the arrays that
describe a scene (geometry, materials, lights, camera rig, image size, depth).
Both sides of the parity check -- `oracle/` (test infrastructure) and the C-ABI
library -- consume exactly these arrays; neither imports the other.

Every floating-point value is rounded to float32 (and stored in float64 arrays)
so the double-precision oracle and the FP32 device path see bit-identical
geometry.

Recipes follow SURVEY.md §8(d) (configs C1..C5 of BASELINE.json) and SPEC.md
scene-model (builtin_object S:82-90, paper_scene S:92-100, default rig S:112,
S:493).  All randomness comes from numpy `Generator(PCG64(seed))`.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

# Material row layout: kd[3], ks[3], shininess, kr, kt, ior  (10 values)
MAT_FIELDS = 10


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def material(kd, ks, shininess=1.0, kr=0.0, kt=0.0, ior=1.0):
    kd = np.broadcast_to(np.asarray(kd, dtype=np.float64), (3,))
    ks = np.broadcast_to(np.asarray(ks, dtype=np.float64), (3,))
    return _f32(np.concatenate([kd, ks, [shininess, kr, kt, ior]]))


# SURVEY.md §8(d) material palette
def M0_plane():
    return material(0.6, 0.0, 1.0, kr=0.25)


def M1_diffuse(kd):
    return material(kd, 0.2, 16.0)


def M2_mirror():
    return material(0.05, 0.8, 128.0, kr=0.8)


def M3_glass():
    return material(0.0, 0.6, 256.0, kr=0.1, kt=0.85, ior=1.5)


def M4_mesh():
    return material((0.7, 0.6, 0.4), 0.3, 32.0, kr=0.3)


@dataclass
class Rig:
    """Stereo rig parameters as passed to rt_set_stereo_camera (north star)."""
    eye: np.ndarray          # cyclopean midpoint
    look_at: np.ndarray
    up: np.ndarray
    vfov_deg: float
    interocular: float
    convergence: float       # <= 0 or inf -> parallel rig

    def as_tuple(self):
        return (self.eye, self.look_at, self.up, self.vfov_deg, self.interocular, self.convergence)


@dataclass
class Scene:
    name: str
    spheres: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    sphere_mat: np.ndarray = field(default_factory=lambda: np.zeros((0,), np.uint32))
    planes: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    plane_mat: np.ndarray = field(default_factory=lambda: np.zeros((0,), np.uint32))
    vertices: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    tris: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.uint32))
    tri_mat: np.ndarray = field(default_factory=lambda: np.zeros((0,), np.uint32))
    materials: np.ndarray = field(default_factory=lambda: np.zeros((0, MAT_FIELDS)))
    lights: np.ndarray = field(default_factory=lambda: np.zeros((0, 6)))
    ambient: np.ndarray = field(default_factory=lambda: np.zeros(3))
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    rig: Rig | None = None
    width: int = 64
    height: int = 48
    max_depth: int = 1

    def finalize(self):
        """Round every value to float32 and fix dtypes/shapes."""
        self.spheres = _f32(self.spheres).reshape(-1, 4)
        self.planes = _f32(self.planes).reshape(-1, 4)
        self.vertices = _f32(self.vertices).reshape(-1, 3)
        self.materials = _f32(self.materials).reshape(-1, MAT_FIELDS)
        self.lights = _f32(self.lights).reshape(-1, 6)
        self.ambient = _f32(self.ambient).reshape(3)
        self.background = _f32(self.background).reshape(3)
        self.sphere_mat = np.ascontiguousarray(self.sphere_mat, dtype=np.uint32).reshape(-1)
        self.plane_mat = np.ascontiguousarray(self.plane_mat, dtype=np.uint32).reshape(-1)
        self.tris = np.ascontiguousarray(self.tris, dtype=np.uint32).reshape(-1, 3)
        self.tri_mat = np.ascontiguousarray(self.tri_mat, dtype=np.uint32).reshape(-1)
        if self.rig is not None:
            r = self.rig
            self.rig = Rig(_f32(r.eye).reshape(3), _f32(r.look_at).reshape(3), _f32(r.up).reshape(3),
                           float(np.float32(r.vfov_deg)), float(np.float32(r.interocular)),
                           float(np.float32(r.convergence)))
        return self

    @property
    def n_spheres(self):
        return len(self.spheres)

    @property
    def n_planes(self):
        return len(self.planes)

    @property
    def n_tris(self):
        return len(self.tris)

    @property
    def n_prims(self):
        return self.n_spheres + self.n_planes + self.n_tris

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.spheres, self.sphere_mat, self.planes, self.plane_mat, self.vertices,
                  self.tris, self.tri_mat, self.materials, self.lights, self.ambient, self.background):
            h.update(np.ascontiguousarray(a).tobytes())
        if self.rig is not None:
            for a in self.rig.as_tuple():
                h.update(np.asarray(a, np.float64).tobytes())
        h.update(f"{self.width}x{self.height}d{self.max_depth}".encode())
        return h.hexdigest()

    def with_view(self, width=None, height=None, max_depth=None, rig=None, name=None):
        """Same geometry, different image size / depth / rig (shares arrays)."""
        s = Scene(**{k: getattr(self, k) for k in self.__dataclass_fields__})
        if width is not None:
            s.width = int(width)
        if height is not None:
            s.height = int(height)
        if max_depth is not None:
            s.max_depth = int(max_depth)
        if rig is not None:
            s.rig = rig
        if name is not None:
            s.name = name
        return s.finalize()


# --------------------------------------------------------------------------------------
# Meshes
# --------------------------------------------------------------------------------------

def torus_mesh(nu, nv, R, r, disp_fn, tilt_deg=30.0):
    """UV torus around the y axis, displaced along the analytic normal, tilted about x.

    u in [0, 2pi) runs around the main ring, v in [0, 2pi) around the tube.
    Two triangles per grid quad, wound counter-clockwise seen from outside
    (SURVEY §8(d) C3/C4 recipe).  Returns (vertices (nu*nv,3), tris (2*nu*nv,3)).
    """
    u = np.arange(nu, dtype=np.float64) * (2.0 * np.pi / nu)
    v = np.arange(nv, dtype=np.float64) * (2.0 * np.pi / nv)
    U, V = np.meshgrid(u, v, indexing="ij")            # (nu, nv)
    nx = np.cos(V) * np.cos(U)
    ny = np.sin(V)
    nz = np.cos(V) * np.sin(U)
    ring = R + r * np.cos(V)
    px = ring * np.cos(U)
    py = r * np.sin(V)
    pz = ring * np.sin(U)
    d = disp_fn(U, V)
    px = px + d * nx
    py = py + d * ny
    pz = pz + d * nz
    t = math.radians(tilt_deg)
    ct, st = math.cos(t), math.sin(t)
    qy = ct * py - st * pz
    qz = st * py + ct * pz
    verts = np.stack([px, qy, qz], axis=-1).reshape(-1, 3)

    i = np.arange(nu)[:, None]
    j = np.arange(nv)[None, :]
    i1 = (i + 1) % nu
    j1 = (j + 1) % nv
    a = (i * nv + j)
    b = (i1 * nv + j)
    c = (i1 * nv + j1)
    dd = (i * nv + j1)
    # orientation: d/du x d/dv points outward for this parameterisation when wound (a, dd, c)
    t0 = np.stack([a, dd, c], axis=-1).reshape(-1, 3)
    t1 = np.stack([a, c, b], axis=-1).reshape(-1, 3)
    tris = np.empty((2 * nu * nv, 3), dtype=np.int64)
    tris[0::2] = t0
    tris[1::2] = t1
    return verts, tris.astype(np.uint32)


def _orient_outward(verts, tris, center):
    v0, v1, v2 = verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]
    n = np.cross(v1 - v0, v2 - v0)
    c = (v0 + v1 + v2) / 3.0 - center
    flip = (n * c).sum(-1) < 0
    out = tris.copy()
    out[flip, 1], out[flip, 2] = tris[flip, 2], tris[flip, 1]
    return out


def builtin_object(kind, center=(0.0, 0.0, 0.0), scale=1.0):
    """SPEC builtin_object: cube (8v/12f), icosahedron (12v/20f), dodeca36 (20v/36f).

    Returns (vertices, tris) with outward (CCW-from-outside) faces.
    """
    from scipy.spatial import ConvexHull

    phi = (1.0 + math.sqrt(5.0)) / 2.0
    if kind == "cube":
        pts = np.array([[x, y, z] for x in (-0.5, 0.5) for y in (-0.5, 0.5) for z in (-0.5, 0.5)])
    elif kind == "icosahedron":
        pts = []
        for s1 in (-1, 1):
            for s2 in (-1, 1):
                pts += [[0, s1, s2 * phi], [s1, s2 * phi, 0], [s2 * phi, 0, s1]]
        pts = np.array(pts, dtype=np.float64) / (2.0 * phi)
    elif kind == "dodeca36":
        pts = [[x, y, z] for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)]
        ip = 1.0 / phi
        for s1 in (-1, 1):
            for s2 in (-1, 1):
                pts += [[0, s1 * ip, s2 * phi], [s1 * ip, s2 * phi, 0], [s2 * phi, 0, s1 * ip]]
        pts = np.array(pts, dtype=np.float64) / (2.0 * phi)
    else:
        raise ValueError(f"unknown builtin object {kind!r}")
    hull = ConvexHull(pts)
    tris = _orient_outward(pts, np.asarray(hull.simplices, dtype=np.int64), np.zeros(3))
    verts = pts * float(scale) + np.asarray(center, dtype=np.float64)
    return verts, tris.astype(np.uint32)


def _merge_meshes(parts):
    verts, tris, mats = [], [], []
    base = 0
    for v, t, m in parts:
        verts.append(v)
        tris.append(t.astype(np.int64) + base)
        mats.append(np.full(len(t), m, np.uint32))
        base += len(v)
    if not verts:
        return np.zeros((0, 3)), np.zeros((0, 3), np.uint32), np.zeros(0, np.uint32)
    return np.concatenate(verts), np.concatenate(tris).astype(np.uint32), np.concatenate(mats)


# --------------------------------------------------------------------------------------
# Configs C1..C5 (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------------------

SKY = (0.25, 0.35, 0.55)
DEFAULT_IOD = 0.065


def _rig(eye, look_at, vfov, iod=DEFAULT_IOD, convergence=None, up=(0.0, 1.0, 0.0)):
    eye = np.asarray(eye, np.float64)
    look_at = np.asarray(look_at, np.float64)
    if convergence is None:      # zero parallax at the look-at point (SURVEY §8(c) reading 13)
        convergence = float(np.linalg.norm(look_at - eye))
    return Rig(eye, look_at, np.asarray(up, np.float64), vfov, iod, convergence)


def scene_c1():
    """C1: 64x48, 3 spheres + ground plane, 1 light, depth 1 (BASELINE.json configs[0])."""
    s = Scene("C1")
    s.materials = np.stack([
        M0_plane(),
        M1_diffuse((0.8, 0.15, 0.1)),
        M2_mirror(),
        M1_diffuse((0.1, 0.2, 0.8)),
    ])
    s.spheres = np.array([[-1.5, 1.0, 0.0, 1.0], [0.0, 1.0, -2.0, 1.0], [1.5, 1.0, 0.5, 1.0]])
    s.sphere_mat = np.array([1, 2, 3], np.uint32)
    s.planes = np.array([[0.0, 1.0, 0.0, 0.0]])
    s.plane_mat = np.array([0], np.uint32)
    s.lights = np.array([[5.0, 8.0, 6.0, 1.0, 1.0, 1.0]])
    s.ambient = np.full(3, 0.1)
    s.background = np.array(SKY)
    s.rig = _rig((0.0, 2.5, 8.0), (0.0, 1.0, 0.0), 40.0)
    s.width, s.height, s.max_depth = 64, 48, 1
    return s.finalize()


def scene_c2(seed=2):
    """C2: 640x480, 8x8 grid of diffuse/mirror/glass spheres + plane, 2 lights, depth 5."""
    rng = np.random.Generator(np.random.PCG64(seed))
    s = Scene("C2")
    mats = [M0_plane(), M2_mirror(), M3_glass()]     # 0 plane, 1 mirror, 2 glass, 3.. diffuse
    spheres, smat = [], []
    for i in range(8):
        for j in range(8):
            x = -7.0 + 2.0 * i + rng.uniform(-0.25, 0.25)
            z = -7.0 + 2.0 * j + rng.uniform(-0.25, 0.25)
            r = rng.uniform(0.3, 0.7)
            spheres.append([x, r + 0.01, z, r])
            cls = (i + j) % 3
            if cls == 0:
                mats.append(M1_diffuse(rng.uniform(0.2, 0.9, 3)))
                smat.append(len(mats) - 1)
            elif cls == 1:
                smat.append(1)
            else:
                smat.append(2)
    s.materials = np.stack(mats)
    s.spheres = np.array(spheres)
    s.sphere_mat = np.array(smat, np.uint32)
    s.planes = np.array([[0.0, 1.0, 0.0, 0.0]])
    s.plane_mat = np.array([0], np.uint32)
    s.lights = np.array([[-8.0, 12.0, 8.0, 0.7, 0.7, 0.7], [10.0, 9.0, -4.0, 0.5, 0.45, 0.4]])
    s.ambient = np.full(3, 0.1)
    s.background = np.array(SKY)
    s.rig = _rig((0.0, 5.0, 16.0), (0.0, 0.0, 0.0), 45.0)
    s.width, s.height, s.max_depth = 640, 480, 5
    return s.finalize()


FOUR_LIGHTS = np.array([[sx * 10.0, 12.0, sz * 10.0, 0.35, 0.35, 0.35]
                        for sx in (-1, 1) for sz in (-1, 1)])


def _torus_box(verts):
    return verts.min(0), verts.max(0)


def scene_c3(seed=3):
    """C3: 1920x1080, 10k-tri displaced torus (M4) + 100 spheres, 4 lights, depth 4."""
    rng = np.random.Generator(np.random.PCG64(seed))
    s = Scene("C3")
    verts, tris = torus_mesh(100, 50, 3.0, 1.0,
                             lambda u, v: 0.08 * np.sin(7 * u) * np.sin(5 * v))
    mats = [M4_mesh(), M2_mirror(), M3_glass()]   # 0 mesh, 1 mirror, 2 glass, 3.. diffuse
    lo, hi = _torus_box(verts)
    spheres, smat = [], []
    while len(spheres) < 100:
        c = rng.uniform([-9.0, -3.0, -9.0], [9.0, 5.0, 9.0])
        r = rng.uniform(0.25, 0.6)
        # not overlapping the torus bounding box
        q = np.clip(c, lo, hi)
        if np.linalg.norm(c - q) <= r + 0.05:
            continue
        if any(np.linalg.norm(c - np.array(o[:3])) <= r + o[3] + 0.05 for o in spheres):
            continue
        spheres.append([c[0], c[1], c[2], r])
        u = rng.uniform()
        if u < 0.4:
            mats.append(M1_diffuse(rng.uniform(0.2, 0.9, 3)))
            smat.append(len(mats) - 1)
        elif u < 0.7:
            smat.append(1)
        else:
            smat.append(2)
    s.materials = np.stack(mats)
    s.spheres = np.array(spheres)
    s.sphere_mat = np.array(smat, np.uint32)
    s.vertices = verts
    s.tris = tris
    s.tri_mat = np.zeros(len(tris), np.uint32)
    s.lights = FOUR_LIGHTS.copy()
    s.ambient = np.full(3, 0.08)
    s.background = np.array(SKY)
    s.rig = _rig((0.0, 4.0, 14.0), (0.0, 0.0, 0.0), 50.0)
    s.width, s.height, s.max_depth = 1920, 1080, 4
    return s.finalize()


def c4_torus(nu=1000, nv=500):
    return torus_mesh(nu, nv, 3.0, 1.0,
                      lambda u, v: 0.05 * np.sin(23 * u) * np.sin(17 * v) + 0.02 * np.sin(61 * u + 3 * v))


def scene_c4(seed=4, nu=1000, nv=500):
    """C4: 1920x1080, 1M-tri displaced torus (M4), 4 lights, depth 4 (the bench workload)."""
    s = Scene("C4" if (nu, nv) == (1000, 500) else f"C4[{nu}x{nv}]")
    verts, tris = c4_torus(nu, nv)
    s.materials = np.stack([M4_mesh()])
    s.vertices = verts
    s.tris = tris
    s.tri_mat = np.zeros(len(tris), np.uint32)
    s.lights = FOUR_LIGHTS.copy()
    s.ambient = np.full(3, 0.08)
    s.background = np.array(SKY)
    s.rig = _rig((0.0, 3.0, 8.0), (0.0, 0.0, 0.0), 50.0)
    s.width, s.height, s.max_depth = 1920, 1080, 4
    return s.finalize()


def c5_rig(k):
    """C5 orbit: eye_k = (8.5 cos th, 3, 8.5 sin th), th = 2 pi k / 240, convergence 8.5."""
    th = 2.0 * math.pi * k / 240.0
    return _rig((8.5 * math.cos(th), 3.0, 8.5 * math.sin(th)), (0.0, 0.0, 0.0), 50.0, convergence=8.5)


def scene_c5(seed=5, frame=0):
    """C5: C4 scene, 3840x2160, depth 6, camera orbit frame `frame` of 60."""
    s = scene_c4(seed)
    s.name = f"C5f{frame}"
    s.rig = c5_rig(frame)
    s.width, s.height, s.max_depth = 3840, 2160, 6
    return s.finalize()


def paper_scene(n_objects):
    """SPEC paper_scene: 1/2/3/5/6 builtin polyhedra + 1 light, fixed layout.

    Layout per SPEC S:112: objects fit a 10x10x10 box centred at the origin,
    camera at z=+15 looking at the origin.
    """
    kinds = {1: ["cube"], 2: ["cube", "icosahedron"], 3: ["cube", "icosahedron", "dodeca36"],
             5: ["cube", "cube", "icosahedron", "icosahedron", "dodeca36"],
             6: ["cube", "icosahedron", "dodeca36", "cube", "icosahedron", "dodeca36"]}
    if n_objects not in kinds:
        raise ValueError("UnsupportedCount")
    ks = kinds[n_objects]
    s = Scene(f"paper{n_objects}")
    parts = []
    mats = []
    for i, k in enumerate(ks):
        ang = 2.0 * math.pi * i / len(ks)
        rad = 0.0 if len(ks) == 1 else 3.0
        c = (rad * math.cos(ang), 0.6 * math.sin(1.7 * i), rad * math.sin(ang))
        v, t = builtin_object(k, c, 2.2)
        hue = [(0.8, 0.3, 0.2), (0.2, 0.7, 0.3), (0.3, 0.4, 0.85), (0.8, 0.7, 0.2), (0.6, 0.3, 0.7),
               (0.3, 0.7, 0.7)][i]
        mats.append(material(hue, 0.3, 24.0, kr=0.2))
        parts.append((v, t, i))
    s.vertices, s.tris, s.tri_mat = _merge_meshes(parts)
    s.materials = np.stack(mats)
    s.lights = np.array([[5.0, 8.0, 10.0, 1.0, 1.0, 1.0]])
    s.ambient = np.full(3, 0.1)
    s.background = np.zeros(3)
    s.rig = _rig((0.0, 0.0, 15.0), (0.0, 0.0, 0.0), 40.0)
    s.width, s.height, s.max_depth = 64, 64, 3
    return s.finalize()


def scene_urchin(n=30000, seed=7):
    """Stress scene for the traversal stack (not a BASELINE config): n triangles radiating from
    the origin in seeded random directions (one vertex within 0.05 of the origin, the other two
    ~2-3 units out and 0.5-1 apart, aspect ratio <= ~6), so every BVH box contains the centre and
    a ray through the centre hits all four children at every level of its first descent: stack
    depth ~3 per BVH4 level, beyond the 16 shared-memory entries.  Mirror-ish material, one light,
    depth 1.  (Slivers 0.01-0.03 wide were tried first: Moller-Trumbore's FP32 edge decision
    degrades with the aspect ratio -- det ~ area, so the barycentric error grows ~aspect x ulp --
    and one shadow ray 2e-4 relative from a sliver's tip edge flipped, outside every band of
    reading 22; the north star's tolerances presume well-shaped triangles like C3/C4's.)"""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    w = rng.normal(size=(n, 3))
    w -= (w * u).sum(1, keepdims=True) * u                 # a direction perpendicular to u
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    r = rng.uniform(2.0, 3.0, size=(n, 1))
    half = rng.uniform(0.25, 0.5, size=(n, 1))
    a = rng.uniform(-0.05, 0.05, size=(n, 3))
    b = r * u + half * w
    c = r * u - half * w
    s = Scene("urchin")
    s.vertices = np.stack([a, b, c], 1).reshape(-1, 3)
    s.tris = np.arange(3 * n, dtype=np.uint32).reshape(n, 3)
    s.tri_mat = np.zeros(n, np.uint32)
    s.materials = np.stack([material((0.7, 0.5, 0.3), 0.4, 24.0, kr=0.3)])
    s.lights = np.array([[4.0, 6.0, 8.0, 1.0, 1.0, 1.0]])
    s.ambient = np.full(3, 0.1)
    s.background = np.array(SKY)
    s.rig = _rig((0.0, 0.0, 8.0), (0.0, 0.0, 0.0), 40.0)
    s.width, s.height, s.max_depth = 40, 30, 1
    return s.finalize()


CONFIGS = {
    "C1": scene_c1,
    "C2": scene_c2,
    "C3": scene_c3,
    "C4": scene_c4,
    "C5": scene_c5,
}


def make_scene(name, **kw):
    return CONFIGS[name](**kw)


def sample_pixels(width, height, n_per_eye, seed):
    """Seeded pixel sample (eye, px, py) int32 triples for sampled parity / CPU baseline."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for eye in (0, 1):
        idx = rng.choice(width * height, size=min(n_per_eye, width * height), replace=False)
        idx.sort()
        out.append(np.stack([np.full(len(idx), eye), idx % width, idx // width], -1))
    return np.concatenate(out).astype(np.int32)
