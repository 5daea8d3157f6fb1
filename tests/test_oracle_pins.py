"""Pins of the CPU oracle (oracle/whitted_oracle.c) against things other than itself:
SPEC worked examples (tests/golden/spec_examples.json), closed forms, invariants and
independent brute force.  CPU only.

Each test names the passage it pins.  P:NN = PAPER.md line, S:NN = SPEC.md line,
R#n = DESIGN.md reading n.
"""
import math

import numpy as np
import pytest

from oracle.oracle import FRAG_BOUNDARY, FRAG_UNSTABLE, Oracle, half_bits
from paper_1702_01530_b200 import scenes
from paper_1702_01530_b200.scenes import Rig, Scene, material

SQ2 = math.sqrt(2.0)


def mk_scene(spheres=(), planes=(), verts=(), tris=(), mats=None, sphere_mat=None, plane_mat=None,
             tri_mat=None, lights=(), ambient=(0, 0, 0), background=(0, 0, 0), rig=None, w=8, h=6, depth=0,
             round32=False):
    s = Scene("t")
    s.spheres = np.asarray(spheres, np.float64).reshape(-1, 4)
    s.planes = np.asarray(planes, np.float64).reshape(-1, 4)
    s.vertices = np.asarray(verts, np.float64).reshape(-1, 3)
    s.tris = np.asarray(tris, np.uint32).reshape(-1, 3)
    s.materials = np.asarray(mats if mats is not None else [material(0.5, 0.0)], np.float64).reshape(-1, 10)
    s.sphere_mat = np.asarray(sphere_mat if sphere_mat is not None else [0] * len(s.spheres), np.uint32)
    s.plane_mat = np.asarray(plane_mat if plane_mat is not None else [0] * len(s.planes), np.uint32)
    s.tri_mat = np.asarray(tri_mat if tri_mat is not None else [0] * len(s.tris), np.uint32)
    s.lights = np.asarray(lights, np.float64).reshape(-1, 6)
    s.ambient = np.asarray(ambient, np.float64) * np.ones(3)
    s.background = np.asarray(background, np.float64) * np.ones(3)
    s.rig = rig or Rig(np.array([0.0, 0, 5]), np.zeros(3), np.array([0.0, 1, 0]), 40.0, 0.0, 0.0)
    s.width, s.height, s.max_depth = w, h, depth
    if round32:
        s.finalize()
    return s


# ----------------------------------------------------------------------------- camera
def test_primary_ray_spec_examples(golden):
    """S:166-167 (generate_primary_ray)."""
    g = golden["primary_ray_1x1"]
    o = Oracle(mk_scene())
    rig = Rig(np.array(g["eye"]), np.array(g["look_at"]), np.array(g["up"]), g["vfov"], 0.0, 0.0)
    cam = o.camera(rig, 1, 1)
    org, d = o.primary_ray(cam, 0, 0, 0)
    axis = np.array(g["look_at"]) - np.array(g["eye"])
    np.testing.assert_allclose(d, axis / np.linalg.norm(axis), atol=1e-15)
    np.testing.assert_allclose(org, g["eye"], atol=0)
    g = golden["primary_ray_2x2"]
    rig = Rig(np.array(g["eye"]), np.array(g["look_at"]), np.array(g["up"]), g["vfov"], 0.0, 0.0)
    cam = o.camera(rig, g["width"], g["height"])
    _, d = o.primary_ray(cam, 0, g["px"], g["py"])
    e = np.array(g["expect_dir_unnormalized"])
    np.testing.assert_allclose(d, e / np.linalg.norm(e), atol=1e-15)


def test_derive_eyes_spec(golden):
    """S:428-430 (derive_eyes): positions, midpoint = base, distance = separation."""
    g = golden["derive_eyes"]
    o = Oracle(mk_scene())
    rig = Rig(np.zeros(3), np.array([0.0, 0, -1]), np.array([0.0, 1, 0]), 60.0, g["sep"], 0.0)
    cam = o.camera(rig, 4, 4)
    np.testing.assert_allclose(cam.eye[0][:], g["left"], atol=1e-17)
    np.testing.assert_allclose(cam.eye[1][:], g["right"], atol=1e-17)
    rng = np.random.default_rng(0)
    for _ in range(100):
        e = rng.normal(size=3) * 5
        la = e + rng.normal(size=3) * 3
        sep = rng.uniform(0.01, 0.2)
        cam = o.camera(Rig(e, la, np.array([0.0, 1, 0]), 50.0, sep, 0.0), 4, 4)
        L, R = np.array(cam.eye[0][:]), np.array(cam.eye[1][:])
        np.testing.assert_allclose((L + R) / 2, e, atol=1e-12)
        assert abs(np.linalg.norm(R - L) - sep) < 1e-12


def test_convergence_closed_form():
    """R#13 off-axis rig: the left-eye ray of image coordinate sx crosses the cyclopean
    axis at depth z = (s/2) / (sx + s/(2C)), i.e. sx_L = s/(2z) - s/(2C) (zero parallax at C);
    the parallel rig (C <= 0) gives parallel centre rays."""
    o = Oracle(mk_scene())
    s, Cv, W, H = 0.3, 6.0, 101, 51
    rig = Rig(np.array([0.0, 0, 0]), np.array([0.0, 0, -1]), np.array([0.0, 1, 0]), 40.0, s, Cv)
    cam = o.camera(rig, W, H)
    th = math.tan(math.radians(20.0))
    for px in (50, 55, 70, 90):
        sx = (2 * (px + 0.5) / W - 1) * th * (W / H)
        for eye, sgn in ((0, -1), (1, +1)):
            org, d = o.primary_ray(cam, eye, px, 25)
            # independent closed form: eye at sgn*s/2 on x, image-plane point (sx + sigma, 0, -1)
            sig = -sgn * s / (2 * Cv)
            np.testing.assert_allclose(org, [sgn * s / 2, 0, 0], atol=1e-15)
            dd = np.array([sx + sig, 0.0, -1.0])
            np.testing.assert_allclose(d, dd / np.linalg.norm(dd), atol=1e-15)
    # centre pixel: both eyes' rays meet at depth C on the axis
    _, dl = o.primary_ray(cam, 0, 50, 25)
    zL = (s / 2) / (dl[0] / -dl[2])
    assert abs(zL - Cv) < 1e-12
    cam = o.camera(Rig(np.zeros(3), np.array([0.0, 0, -1]), np.array([0.0, 1, 0]), 40.0, s, 0.0), W, H)
    _, dl = o.primary_ray(cam, 0, 50, 25)
    _, dr = o.primary_ray(cam, 1, 50, 25)
    np.testing.assert_allclose(dl, dr, atol=0)
    np.testing.assert_allclose(dl, [0, 0, -1], atol=1e-15)


# ----------------------------------------------------------------------------- primitives
def test_ray_sphere_closed_form():
    """Ray (h,0,0) + t(0,0,-1) vs sphere c=(0,0,-10), r=2: t = 10 - sqrt(4 - h^2), miss for |h|>2;
    origin at the centre -> t = r (SURVEY §8(c) pin table)."""
    o = Oracle(mk_scene(spheres=[[0, 0, -10, 2]]))
    for h in np.linspace(-1.99, 1.99, 41):
        t, pid = o.nearest([h, 0, 0], [0, 0, -1])
        assert pid == 0
        assert abs(t - (10 - math.sqrt(4 - h * h))) < 1e-12
    for h in (2.01, -2.5, 3.0):
        t, pid = o.nearest([h, 0, 0], [0, 0, -1])
        assert pid == -1 and math.isinf(t)
    t, pid = o.nearest([0, 0, -10], [0, 0.6, 0.8])
    assert pid == 0 and abs(t - 2.0) < 1e-12


def test_ray_plane_closed_form():
    """Ray (0,2,0), d = (1,-1,0)/sqrt2 vs y=0: t = 2 sqrt2; n.d = 0 -> miss."""
    o = Oracle(mk_scene(planes=[[0, 1, 0, 0]]))
    t, pid = o.nearest([0, 2, 0], [1 / SQ2, -1 / SQ2, 0])
    assert pid == 0 and abs(t - 2 * SQ2) < 1e-12
    t, pid = o.nearest([0, 2, 0], [1, 0, 0])
    assert pid == -1
    t, pid = o.nearest([0, 2, 0], [0, 1, 0])        # plane behind the ray
    assert pid == -1


def test_triangle_spec_examples(golden):
    """S:176-178 (intersect_triangle) and S:187 (stacked triangles -> nearest)."""
    g = golden["triangle"]
    o = Oracle(mk_scene(verts=g["v"], tris=[[0, 1, 2]]))
    for c in g["cases"]:
        t, pid = o.nearest(c["o"], c["d"])
        if c["t"] is None:
            assert pid == -1
        else:
            assert pid == 0 and t == c["t"]
    v = np.array(g["v"], float)
    v7 = v.copy()
    v7[:, 2] = 7
    o = Oracle(mk_scene(verts=np.concatenate([v7, v]), tris=[[0, 1, 2], [3, 4, 5]]))
    t, pid = o.nearest([0, 0, 0], [0, 0, 1])
    assert t == golden["stacked"]["t_near"] and pid == 1


def test_shared_edge_tie_goes_to_smaller_id():
    """S:300 (query_nearest): a ray through the shared edge of two faces -> smaller index (R#9)."""
    verts = [[0, 0, 5], [1, 0, 5], [0, 1, 5], [1, 1, 5]]
    o = Oracle(mk_scene(verts=verts, tris=[[1, 3, 2], [0, 1, 2]]))
    t, pid = o.nearest([0.5, 0.5, 0], [0, 0, 1])        # on the diagonal edge (1,0)-(0,1)
    assert pid == 0 and t == 5.0
    o = Oracle(mk_scene(verts=verts, tris=[[0, 1, 2], [1, 3, 2]]))
    assert o.nearest([0.5, 0.5, 0], [0, 0, 1])[1] == 0
    # sphere (ID 0) tangent-touching a triangle at the same t: sphere wins by ID order
    o = Oracle(mk_scene(spheres=[[0.25, 0.25, 6, 1]], verts=verts, tris=[[0, 1, 2]]))
    t, pid = o.nearest([0.25, 0.25, 0], [0, 0, 1])
    assert pid == 0 and t == 5.0


def _np_nearest(scene, o, d, tmin=1e-4):
    """Independent brute force: triangles via np.linalg.solve of [-d e1 e2][t u v] = o - v0,
    spheres via the geometric chord form, planes via the point-normal form."""
    best, bid = np.inf, -1
    gid = 0
    for c in scene.spheres:
        ctr, r = c[:3], c[3]
        tc = np.dot(ctr - o, d)
        D2 = np.dot(ctr - o, ctr - o) - tc * tc
        if D2 <= r * r:
            hc = math.sqrt(r * r - D2)
            for t in (tc - hc, tc + hc):
                if t > tmin:
                    if t < best:
                        best, bid = t, gid
                    break
        gid += 1
    for p in scene.planes:
        n = p[:3]
        pt = n * p[3] / np.dot(n, n)
        den = np.dot(n, d)
        if den != 0:
            t = np.dot(pt - o, n) / den
            if t > tmin and t < best:
                best, bid = t, gid
        gid += 1
    for tri in scene.tris:
        v0, v1, v2 = scene.vertices[tri]
        A = np.stack([-d, v1 - v0, v2 - v0], 1)
        if abs(np.linalg.det(A)) > 1e-14:
            t, u, v = np.linalg.solve(A, o - v0)
            if u >= 0 and v >= 0 and u + v <= 1 and t > tmin and t < best:
                best, bid = t, gid
        gid += 1
    return best, bid


def test_nearest_vs_independent_bruteforce():
    """S:222 nearest-hit exhaustiveness / S:183 tie-break: oracle vs an independent numpy
    all-pairs minimum on random tiny scenes (<= 8 prims)."""
    rng = np.random.default_rng(7)
    mism = 0
    for trial in range(30):
        ns, npl, nt = rng.integers(0, 3), rng.integers(0, 2), rng.integers(1, 5)
        sph = np.concatenate([rng.uniform(-2, 2, (ns, 3)), rng.uniform(0.3, 1.0, (ns, 1))], 1)
        pl = np.concatenate([rng.normal(size=(npl, 3)), rng.uniform(-3, -1, (npl, 1))], 1)
        verts = rng.uniform(-2, 2, (3 * nt, 3))
        tris = np.arange(3 * nt).reshape(-1, 3)
        s = mk_scene(spheres=sph, planes=pl, verts=verts, tris=tris)
        o = Oracle(s)
        for _ in range(40):
            org = rng.uniform(-4, 4, 3)
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            t, pid = o.nearest(org, d)
            t2, pid2 = _np_nearest(s, org, d)
            if pid != pid2:
                mism += 1
                continue
            if pid >= 0:
                assert abs(t - t2) <= 1e-9 * max(1, t)
    assert mism == 0


# ----------------------------------------------------------------------------- shading
def test_shade_spec_examples(golden):
    """S:196-197 (shade) and S:206-207 (trace)."""
    # a triangle facing +z at z=0, viewed head-on, light straight along the normal
    verts = [[-5, -5, 0], [5, -5, 0], [0, 5, 0]]
    light = [[0, 0, 10, 1, 1, 1]]
    s = mk_scene(verts=verts, tris=[[0, 1, 2]], mats=[material(0.5, 0.0)], lights=light)
    rgb, cnt = Oracle(s).trace_ray([0, 0, 3], [0, 0, -1], 0)
    np.testing.assert_allclose(rgb, golden["shade_diffuse"]["expect"], atol=1e-15)
    assert cnt[3] == 1
    # occluder between point and light -> ambient*kd only
    sv = verts + [[-1, -1, 5], [1, -1, 5], [0, 1, 5]]
    s = mk_scene(verts=sv, tris=[[0, 1, 2], [3, 4, 5]], mats=[material(0.5, 0.0)], lights=light,
                 ambient=0.2)
    rgb, _ = Oracle(s).trace_ray([0, 0.2, 3], [0, 0, -1], 0)
    np.testing.assert_allclose(rgb, [0.1, 0.1, 0.1], atol=1e-15)
    # empty scene -> background
    g = golden["trace_empty"]
    rgb, _ = Oracle(mk_scene(background=g["background"])).trace_ray([0, 0, 0], [0, 0, 1], 3)
    np.testing.assert_allclose(rgb, g["background"], atol=0)
    # pure-ambient surface
    s = mk_scene(verts=verts, tris=[[0, 1, 2]], mats=[material(1.0, 0.0)], ambient=0.1)
    rgb, _ = Oracle(s).trace_ray([0, 0, 3], [0, 0, -1], 2)
    np.testing.assert_allclose(rgb, golden["trace_ambient"]["expect"], atol=1e-16)


def test_analytic_single_sphere_image():
    """Analytic single-sphere image (SURVEY §8(c) pin): unit sphere at the origin, eyes at
    (+-s/2, 0, 5), light (3,3,5), kd (0.8,0.5,0.3), ks 0.5, n 20, ambient 0.1, bg 0.
    Convex and alone, so no shadowing where n.l > 0.  Closed form per pixel in numpy
    (chord form of the hit, Phong with reflect vector), rim pixels (F2-F4) excluded."""
    W, H, s, Cv = 48, 40, 0.2, 5.0
    kd, ks, n, amb = np.array([0.8, 0.5, 0.3]), 0.5, 20.0, 0.1
    L = np.array([3.0, 3.0, 5.0])
    rig = Rig(np.array([0.0, 0, 5]), np.zeros(3), np.array([0.0, 1, 0]), 40.0, s, Cv)
    sc = mk_scene(spheres=[[0, 0, 0, 1]], mats=[material(kd, ks, n)], lights=[[3, 3, 5, 1, 1, 1]],
                  ambient=amb, rig=rig, w=W, h=H, depth=0)
    out = Oracle(sc).render()
    th = math.tan(math.radians(20))
    checked = 0
    for eye, sgn in ((0, -1), (1, 1)):
        e = np.array([sgn * s / 2, 0, 5.0])
        sig = -sgn * s / (2 * Cv)
        for py in range(H):
            for px in range(W):
                sx = (2 * (px + 0.5) / W - 1) * th * W / H
                sy = (1 - 2 * (py + 0.5) / H) * th
                d = np.array([sx + sig, sy, -1.0])
                d /= np.linalg.norm(d)
                tc = -np.dot(e, d)
                D2 = np.dot(e, e) - tc * tc
                got = out["radiance"][eye, py, px]
                if out["pflags"][eye, py, px]:
                    continue
                if D2 > 1:
                    np.testing.assert_allclose(got, 0, atol=0)
                    assert out["id"][eye, py, px] == -1
                    continue
                p = e + (tc - math.sqrt(1 - D2)) * d
                nn = p / np.linalg.norm(p)
                l = (L - p) / np.linalg.norm(L - p)
                ndl = np.dot(nn, l)
                c = amb * kd
                if ndl > 0:
                    r = 2 * ndl * nn - l
                    c = c + kd * ndl + ks * max(0.0, np.dot(r, -d)) ** n
                np.testing.assert_allclose(got, c, atol=1e-12)
                assert out["id"][eye, py, px] == 0
                checked += 1
    assert checked > 400


def test_ground_plane_under_light():
    """Plane y=0 under a light at height h: radiance = ambient*kd + kd*I*h/|L-q| + ks*I*(r.v)^n
    with r the mirror of l (closed form at a hit point q)."""
    h, kd, ks, n = 4.0, 0.6, 0.3, 8.0
    s = mk_scene(planes=[[0, 1, 0, 0]], mats=[material(kd, ks, n)], lights=[[1, h, 0, 1, 1, 1]], ambient=0.05)
    org = np.array([-3.0, 3.0, 0.0])
    d = np.array([1.0, -1.0, 0.0]) / SQ2                    # hits q = (0,0,0)
    rgb, _ = Oracle(s).trace_ray(org, d, 0)
    Lq = np.array([1.0, h, 0.0])
    l = Lq / np.linalg.norm(Lq)
    r = np.array([-l[0], l[1], -l[2]])                        # reflect l about +y: 2(n.l)n - l
    expect = 0.05 * kd + kd * h / np.linalg.norm(Lq) + ks * max(0, np.dot(r, -d)) ** n
    np.testing.assert_allclose(rgb, expect, atol=1e-14)


def test_shadow_monotonicity():
    """removing all occluders never decreases any pixel (2-triangle scene + blocker)."""
    verts = [[-4, -1, -4], [4, -1, -4], [0, -1, 4], [-0.5, 0.5, -0.5], [0.5, 0.5, -0.5], [0, 0.5, 0.5]]
    rig = Rig(np.array([0.0, 3, 6]), np.zeros(3), np.array([0.0, 1, 0]), 50.0, 0.065, 0.0)
    kw = dict(verts=verts, mats=[material(0.7, 0.3, 10)], lights=[[0, 6, 0, 1, 1, 1], [3, 4, 2, 0.5, 0.4, 0.3]],
              ambient=0.1, rig=rig, w=24, h=16, depth=2)
    with_b = Oracle(mk_scene(tris=[[0, 2, 1], [3, 5, 4]], **kw)).render()
    floor_only = Oracle(mk_scene(tris=[[0, 2, 1]], **kw)).render()
    m = (with_b["id"] == 0) & (with_b["tflags"] == 0) & (floor_only["tflags"] == 0)
    assert m.sum() > 50
    assert np.all(floor_only["radiance"][m] >= with_b["radiance"][m] - 1e-15)
    assert np.any(floor_only["radiance"][m] > with_b["radiance"][m] + 1e-3)   # some shadow existed


def test_facing_mirrors_recursion_count(golden):
    """two facing mirrors, max_depth 3 -> exactly 3 reflection recursions."""
    g = golden["facing_mirrors"]
    s = mk_scene(planes=[[0, 0, 1, -1], [0, 0, 1, 1]], mats=[material(0.0, 0.0, 1, kr=1.0)])
    for depth in (0, 1, 3, 7):
        _, cnt = Oracle(s).trace_ray([0, 0, 0], [0, 0, 1], depth)
        assert cnt[1] == depth
    _, cnt = Oracle(s).trace_ray([0, 0, 0], [0, 0, 1], g["max_depth"])
    assert cnt[1] == g["reflections"]


def test_reflect_spec_examples():
    """S:216-217 (reflect): d = normalize(1,-1,0) about +y -> normalize(1,1,0); normal incidence
    returns straight back.  Observed through what the reflected ray hits: a mirror plane y=0
    (kd=ks=0, kr=1) and a small emissive-free diffuse target lit by ambient only."""
    tgt = [[4.0, 2.0, 0.0, 0.3]]                               # on the line (2,0,0) + t(1,1,0)/sqrt2
    mats = [material(1.0, 0.0), material(0.0, 0.0, 1, kr=1.0)]
    s = mk_scene(spheres=tgt, planes=[[0, 1, 0, 0]], mats=mats, sphere_mat=[0], plane_mat=[1],
                 ambient=0.5, background=0.0)
    rgb, cnt = Oracle(s).trace_ray([0, 2, 0], [1 / SQ2, -1 / SQ2, 0], 1)
    np.testing.assert_allclose(rgb, 0.5, atol=1e-15)
    assert cnt[1] == 1
    # mirror facing -z, target behind the ray origin: normal incidence returns along +z
    s = mk_scene(spheres=[[0, 0, 3, 0.5]], planes=[[0, 0, 1, -2]], mats=mats, sphere_mat=[0], plane_mat=[1],
                 ambient=0.5, background=0.0)
    rgb, _ = Oracle(s).trace_ray([0, 0, 1], [0, 0, -1], 1)
    np.testing.assert_allclose(rgb, 0.5, atol=1e-15)


def test_mirror_sphere_invisible():
    """Perfect mirror sphere (kd=ks=0, kr=1) alone in an empty world shows the background
    at depth >= 1; kr = 0.5 -> 0.5*bg; depth 0 -> black (SURVEY §8(c) pin table)."""
    bg = np.array([0.3, 0.5, 0.7])
    for kr, depth, scale in ((1.0, 1, 1.0), (1.0, 4, 1.0), (0.5, 1, 0.5), (1.0, 0, 0.0)):
        s = mk_scene(spheres=[[0, 0, 0, 1]], mats=[material(0.0, 0.0, 1, kr=kr)], background=bg,
                     w=20, h=16, depth=depth)
        out = Oracle(s).render()
        hit = (out["id"] == 0) & (out["tflags"] == 0)
        assert hit.sum() > 50
        np.testing.assert_allclose(out["radiance"][hit], np.broadcast_to(scale * bg, (hit.sum(), 3)), atol=1e-15)


def test_refraction_index_matched_sphere_invisible():
    """ior = 1, kt = 1, kd = ks = kr = 0 sphere in an empty, light-free world is invisible at
    depth >= 2 (enter + exit): pixels = bg (off-rim); 1e-9 covers the 1e-4 inward bias shift."""
    bg = np.array([0.2, 0.6, 0.4])
    s = mk_scene(spheres=[[0, 0, 0, 1]], mats=[material(0.0, 0.0, 1, kt=1.0, ior=1.0)], background=bg,
                 w=20, h=16, depth=2)
    out = Oracle(s).render()
    hit = (out["id"] == 0) & (out["tflags"] == 0)
    assert hit.sum() > 50
    np.testing.assert_allclose(out["radiance"][hit], np.broadcast_to(bg, (hit.sum(), 3)), atol=1e-9)
    assert out["counts"][2] == 2 * hit.sum() + 2 * ((out["id"] == 0) & (out["tflags"] != 0)).sum()


def test_refraction_snell_and_tir():
    """Snell at one interface: a ray through a glass sphere's centre is undeviated (it reaches
    a target straight behind); TIR onset at sin(theta) = 1/ior from inside (R#5)."""
    mats = [material(0.0, 0.0, 1, kt=1.0, ior=1.5), material(1.0, 0.0)]
    s = mk_scene(spheres=[[0, 0, 0, 1], [0, 0, -5, 0.2]], mats=mats, sphere_mat=[0, 1], ambient=0.7)
    rgb, cnt = Oracle(s).trace_ray([0, 0, 5], [0, 0, -1], 3)
    np.testing.assert_allclose(rgb, 0.7, atol=1e-15)
    assert cnt[2] == 2
    # from inside, hitting the surface at angle theta from the normal
    s = mk_scene(spheres=[[0, 0, 0, 1]], mats=[material(0.0, 0.0, 1, kt=1.0, ior=1.5)])
    crit = math.asin(1 / 1.5)
    for th, refr in ((crit - 0.01, 1), (crit + 0.01, 0), (0.2, 1), (1.2, 0)):
        # start at a point inside and aim at the surface point (0,1,0) so that the angle
        # between -d and the inward normal is theta
        p = np.array([0.0, 1.0, 0.0])
        d = np.array([math.sin(th), math.cos(th), 0.0])
        org = p - 0.5 * d
        _, cnt = Oracle(s).trace_ray(org, d, 1)
        assert cnt[2] == refr and cnt[1] == 1 - refr


# ----------------------------------------------------------------------------- whole-tree invariants
def _c2_small():
    return scenes.scene_c2().with_view(width=40, height=30, max_depth=3)


def test_light_superposition_and_linearity():
    """R(A u B) + R(0) = R(A) + R(B) (unclamped; each light adds a term and shadows are
    per light); scaling every I, ambient and bg by a scales R by a."""
    base = _c2_small()
    A, B = base.lights[:1], base.lights[1:]

    def run(lights, scale=1.0):
        s = base.with_view()
        s.lights = np.concatenate([lights[:, :3], lights[:, 3:] * scale], 1) if len(lights) else lights.reshape(0, 6)
        s.ambient = base.ambient * scale
        s.background = base.background * scale
        return Oracle(s).render(flags=False)["radiance"]

    rab, ra, rb, r0 = run(base.lights), run(A), run(B), run(np.zeros((0, 6)))
    np.testing.assert_allclose(rab + r0, ra + rb, atol=1e-12)
    np.testing.assert_allclose(run(base.lights, 0.37), 0.37 * rab, atol=1e-12)


def test_monotone_in_depth_and_finite():
    """Unclamped R is non-decreasing in max_depth (all terms >= 0); finite everywhere."""
    base = _c2_small()
    prev = None
    for depth in range(0, 5):
        r = Oracle(base.with_view(max_depth=depth)).render(flags=False)["radiance"]
        assert np.all(np.isfinite(r))
        if prev is not None:
            assert np.all(r >= prev - 1e-15)
        prev = r


def _mirror_x(s):
    m = s.with_view()
    m.spheres = s.spheres * [-1, 1, 1, 1]
    m.planes = s.planes * [-1, 1, 1, 1]
    m.vertices = s.vertices * [-1, 1, 1]
    m.tris = s.tris[:, [0, 2, 1]].copy()                      # keep outward normals
    m.lights = s.lights * [-1, 1, 1, 1, 1, 1]
    return m


def test_stereo_mirror_symmetry():
    """Mirror the scene about the rig midplane x=0 (r^ = x^): left(MS) = fliplr(right(S)) and
    right(MS) = fliplr(left(S)), IDs included (north star oracle check)."""
    s = scenes.paper_scene(3)
    c2 = scenes.scene_c2()
    s.spheres = c2.spheres[:12] * [0.5, 0.5, 0.5, 0.5] + [0, -1.5, 0, 0]
    s.sphere_mat = np.zeros(12, np.uint32)
    s = s.with_view(width=32, height=24, max_depth=3,
                    rig=Rig(np.array([0.0, 2.0, 12.0]), np.array([0.0, 0.0, 0.0]), np.array([0.0, 1, 0]),
                            45.0, 0.4, 10.0))
    a = Oracle(s).render()
    b = Oracle(_mirror_x(s)).render()
    for e in (0, 1):
        ok = (a["tflags"][1 - e] == 0) & (b["tflags"][e][:, ::-1] == 0)
        assert ok.mean() > 0.9
        np.testing.assert_allclose(b["radiance"][e][:, ::-1][ok], a["radiance"][1 - e][ok], atol=1e-12)
        okid = (a["pflags"][1 - e] == 0) & (b["pflags"][e][:, ::-1] == 0)
        np.testing.assert_array_equal(b["id"][e][:, ::-1][okid], a["id"][1 - e][okid])
    # separation -> 0 gives identical eyes
    z = Oracle(s.with_view(rig=Rig(s.rig.eye, s.rig.look_at, s.rig.up, 45.0, 0.0, 10.0))).render(flags=False)
    np.testing.assert_array_equal(z["radiance"][0], z["radiance"][1])


# ----------------------------------------------------------------------------- outputs
def test_quantize_rgba8_and_half(golden):
    """S:494 8-bit rounding (half away from zero); RGBA16F = binary16 RNE (R#16), checked
    against numpy's float16 conversion."""
    for c, b in golden["quantize"]["cases"]:
        s = mk_scene(background=c, w=1, h=1)
        out = Oracle(s).render(flags=False)
        assert out["rgba8"][0, 0, 0, 0] == b and out["rgba8"][0, 0, 0, 3] == 255
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.uniform(0, 1, 2000), rng.uniform(0, 1e-4, 200), [0, 1, 2 ** -14, 2 ** -24, 0.5]])
    for x in xs:
        assert half_bits(x) == np.float16(x).view(np.uint16), x


def test_fragility_flags():
    """R#22: a primary ray through a shared mesh edge or a sphere silhouette is flagged;
    a ray through the middle of a face is not."""
    verts = [[-1, -1, 0], [1, -1, 0], [-1, 1, 0], [1, 1, 0]]
    W = H = 5
    rig = Rig(np.array([0.0, 0, 5]), np.zeros(3), np.array([0.0, 1, 0]), 20.0, 0.0, 0.0)
    s = mk_scene(verts=verts, tris=[[0, 1, 2], [1, 3, 2]], rig=rig, w=W, h=H)
    out = Oracle(s).render()
    # centre pixel ray goes through (0,0,0), on the diagonal shared edge
    assert out["pflags"][0, 2, 2] & FRAG_BOUNDARY
    assert out["pflags"][0, 1, 1] == 0 or out["pflags"][0, 3, 1] == 0
    # sphere tangent to the centre pixel's ray (centre (1,0,0), r = 1, ray x = y = 0): silhouette
    out = Oracle(mk_scene(spheres=[[1, 0, 0, 1]], rig=rig, w=W, h=H)).render()
    assert out["pflags"][0, 2, 2] & FRAG_BOUNDARY
    # moved 1e-3 off the silhouette (relative 2e-4 > eps_sphere = 1e-4): robust again
    out = Oracle(mk_scene(spheres=[[1.001, 0, 0, 1]], rig=rig, w=W, h=H)).render()
    assert out["pflags"][0, 2, 2] == 0 and out["id"][0, 2, 2] == -1
    out = Oracle(mk_scene(spheres=[[0.999, 0, 0, 1]], rig=rig, w=W, h=H)).render()
    assert out["pflags"][0, 2, 2] == 0 and out["id"][0, 2, 2] == 0


def _perturbed_dirs(d, delta):
    a = np.array([0.0, 1, 0]) if abs(d[1]) < 0.9 else np.array([1.0, 0, 0])
    u = np.cross(d, a)
    u /= np.linalg.norm(u)
    w = np.cross(d, u)
    return [(d + delta * q) / np.linalg.norm(d + delta * q) for q in (u, -u, w, -w)]


def test_unstable_flag_smooth_scene_never_fires():
    """R#22 (F7): on a lone diffuse sphere the radiance is a smooth function of the ray direction
    away from the silhouette (|dL/dtheta| * 1e-6 << 1e-3), so F7 may only fire on pixels
    that F1-F6 already flag (rim / terminator)."""
    rig = Rig(np.array([0.0, 0, 5]), np.zeros(3), np.array([0.0, 1, 0]), 40.0, 0.2, 5.0)
    sc = mk_scene(spheres=[[0, 0, 0, 1]], mats=[material((0.8, 0.5, 0.3), 0.5, 20)], lights=[[3, 3, 5, 1, 1, 1]],
                  ambient=0.1, rig=rig, w=48, h=40, depth=2)
    out = Oracle(sc).render()
    unstable = (out["tflags"] & FRAG_UNSTABLE) != 0
    assert not np.any(unstable & (out["tflags"] == FRAG_UNSTABLE))
    # F7 off: never set
    out0 = Oracle(sc).render(eps=dict(perturb=0.0))
    assert not np.any(out0["tflags"] & FRAG_UNSTABLE)


def test_unstable_flag_matches_definition():
    """R#22 (F7): in C2 (mirror + glass spheres over a reflective floor, Phong n = 128/256) angular
    error grows at every curved bounce, so some pixels that no structural band (F1-F6) catches
    are unstable.  Check the flag against its definition by tracing the perturbed primaries
    independently (numpy basis, single-ray entry point; four directions at 1e-6, 1e-7 and
    1e-6/33 rad): flagged <=> some clamped channel moves by more than 1e-3."""
    sc = scenes.scene_c2().with_view(width=160, height=120)
    o = Oracle(sc)
    out = o.render()
    tf = out["tflags"]
    only7 = tf == FRAG_UNSTABLE
    assert only7.sum() >= 10, "expected amplification-only unstable pixels"
    cam = o.camera()
    rng = np.random.default_rng(7)
    cand = [tuple(p) for p in np.argwhere(only7)[:20]]
    cand += [(int(rng.integers(2)), int(rng.integers(120)), int(rng.integers(160))) for _ in range(20)]
    for eye, py, px in cand:
        org, d = o.primary_ray(cam, int(eye), int(px), int(py))
        base = np.clip(out["radiance"][eye, py, px], 0, 1)
        moved = max(np.abs(np.clip(o.trace_ray(org, dq, sc.max_depth)[0], 0, 1) - base).max()
                    for delta in (1e-6, 1e-6 * 0.1, 1e-6 / 33.0) for dq in _perturbed_dirs(d, delta))
        assert bool(tf[eye, py, px] & FRAG_UNSTABLE) == (moved > 1e-3), (eye, py, px, moved)


def test_scene_generators(golden):
    """SPEC builtin_object / paper_scene counts and outward torus winding."""
    for k in ("cube", "icosahedron", "dodeca36"):
        nv, nf = golden["builtin_counts"][k]
        v, t = scenes.builtin_object(k)
        assert (len(v), len(t)) == (nv, nf)
        v0, v1, v2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
        nrm = np.cross(v1 - v0, v2 - v0)
        assert np.all((nrm * (v0 + v1 + v2)).sum(1) > 0)
        assert np.all(np.linalg.norm(nrm, axis=1) / 2 > 1e-12)
    assert scenes.paper_scene(5).n_tris == golden["paper_scene5_tris"]["tris"]
    v, t = scenes.torus_mesh(40, 20, 3.0, 1.0, lambda u, w: 0 * u, tilt_deg=0.0)
    v0, v1, v2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    nrm = np.cross(v1 - v0, v2 - v0)
    cen = (v0 + v1 + v2) / 3
    ring = cen.copy()
    ring[:, 1] = 0
    ring = ring / np.linalg.norm(ring, axis=1, keepdims=True) * 3.0
    assert np.all((nrm * (cen - ring)).sum(1) > 0)
    s3 = scenes.scene_c3()
    assert s3.n_tris == 10000 and s3.n_spheres == 100
    assert scenes.scene_c2().n_spheres == 64
    assert scenes.scene_c2().sha256() == scenes.scene_c2().sha256()


def test_refraction_slab_snell_closed_form():
    """Snell's law off-axis (R#5-6): a glass slab (planes y=0 with +y normal, y=-1 with -y
    normal, ior 1.5, kt 1) over a diffuse floor y=-3 lit from (0,-2,0).  A ray from (0,1,0) at
    angle th lands on the floor at x = 3 tan(th) + tan(th_t), sin(th_t) = sin(th)/1.5, where the
    floor radiance is kd*I*n.l = 1/sqrt(1 + x^2).  1e-3 covers the 1e-4 bias offsets."""
    mats = [material(0.0, 0.0, 1, kt=1.0, ior=1.5), material(1.0, 0.0)]
    s = mk_scene(planes=[[0, 1, 0, 0], [0, -1, 0, 1], [0, 1, 0, -3]], mats=mats, plane_mat=[0, 0, 1],
                 lights=[[0, -2, 0, 1, 1, 1]])
    o = Oracle(s)
    for th in (0.1, 0.4, 0.7, 1.0):
        d = np.array([math.sin(th), -math.cos(th), 0.0])
        rgb, cnt = o.trace_ray([0, 1, 0], d, 2)
        tht = math.asin(math.sin(th) / 1.5)
        x = 3 * math.tan(th) + math.tan(tht)
        np.testing.assert_allclose(rgb, 1 / math.sqrt(1 + x * x), atol=1e-3)
        assert cnt[2] == 2
    # kt weighting: kt = 0.5 index-matched sphere -> 0.25 * bg after enter + exit
    bg = np.array([0.2, 0.6, 0.4])
    s = mk_scene(spheres=[[0, 0, 0, 1]], mats=[material(0.0, 0.0, 1, kt=0.5, ior=1.0)], background=bg)
    rgb, _ = Oracle(s).trace_ray([0.1, 0.2, 5], [0, 0, -1], 2)
    np.testing.assert_allclose(rgb, 0.25 * bg, atol=1e-9)


def test_compose_spec_examples(golden):
    """SPEC.md:448-450 (compose_anaglyph) and S:458-460 (compose_sbs) worked examples and
    properties: identical channels -> identity / identical halves; locality."""
    from oracle.oracle import compose
    for case in golden["anaglyph"]["cases"]:
        L = np.array(case["L"] + [255], np.uint8).reshape(1, 1, 4)
        R = np.array(case["R"] + [255], np.uint8).reshape(1, 1, 4)
        np.testing.assert_array_equal(compose(L, R, "anaglyph")[0, 0, :3], case["out"])
    a, b = golden["sbs"]["cols"]
    L = np.array([[[a, a, a, 255], [b, b, b, 255]]], np.uint8)
    out = compose(L, L, "sbs")
    assert out.shape == (1, 2, 4) and np.all(out[0, :, :3] == golden["sbs"]["out"])
    rng = np.random.default_rng(5)
    X = rng.integers(0, 256, (5, 7, 4), dtype=np.uint8)
    X[..., 3] = 255
    np.testing.assert_array_equal(compose(X, X, "anaglyph"), X)
    s = compose(X, X, "sbs")
    assert s.shape == (5, 6, 4)
    np.testing.assert_array_equal(s[:, :3], s[:, 3:])
    # round half up on an odd pair sum; floor(W/2) columns (last column of odd W dropped)
    Y = np.zeros((1, 3, 4), np.uint8)
    Y[0, 0, :3], Y[0, 1, :3], Y[0, 2, :3] = 1, 2, 200
    assert compose(Y, Y, "sbs")[0, 0, 0] == 2
    # locality: one changed input pixel changes exactly one anaglyph pixel
    Z = X.copy()
    Z[2, 3, 0] ^= 0xFF
    d = np.any(compose(Z, X, "anaglyph") != compose(X, X, "anaglyph"), -1)
    assert d.sum() == 1 and d[2, 3]


@pytest.mark.parametrize("cfg,n,depth", [("C1", 100, None), ("C2", 60, None), ("paper3", 40, 3)])
def test_double_precision_adequacy_mpmath(cfg, n, depth):
    """SURVEY §8(c) 'double-precision adequacy': the oracle (double) equals an independent 40-digit
    mpmath evaluation of the same definition (tests/mp_whitted.py: Cramer-rule triangles, written
    from §8(c) steps 1-5) within 1e-9 on seeded non-fragile pixels."""
    from tests import mp_whitted
    sc = scenes.paper_scene(3) if cfg == "paper3" else scenes.make_scene(cfg)
    if depth is not None:
        sc = sc.with_view(max_depth=depth)
    pix = scenes.sample_pixels(sc.width, sc.height, n // 2, seed=11)
    out = Oracle(sc).render(pixels=pix)
    ms = mp_whitted.MpScene(sc)
    checked = 0
    for k, (eye, px, py) in enumerate(pix):
        if out["tflags"][k]:
            continue
        o, d = mp_whitted.primary_ray(sc.rig, sc.width, sc.height, int(eye), int(px), int(py))
        ref = np.array([float(x) for x in ms.trace(o, d, sc.max_depth)])
        np.testing.assert_allclose(out["radiance"][k], ref, atol=1e-9, rtol=0, err_msg=str((eye, px, py)))
        checked += 1
    assert checked >= 0.6 * len(pix)
