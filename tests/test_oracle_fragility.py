"""Pins of the oracle's exclusion classifier (reading 22, the north star's "within 1e-4
relative of a competing hit or of a silhouette") and of its near-tie candidate sets.  CPU only.

Every flag is pinned by a hand-built case whose geometry puts the deciding quantity on either
side of its band (closed form), so a dropped term, a wrong sign or a swapped band fails a test:
  F1 COMPETE  stacked coplanar triangles, separation 0 / 0.5 / 2 x eps_t * t
  F2/F3       shared mesh edge and sphere silhouette (tests/test_oracle_pins.py)
  F4 GRAZE    |n.d| = 5e-5 (flagged) / 2e-4 (not)
  F5 RANGE    a surface at t_min +- 5e-6 (flagged) / +- 5e-5 (not)
  F6 SHADE    n.l = +-5e-5 at the hit; the TIR discriminant k = +-5e-5
  SHADOW      shadow segment 0.5 eps_edge t from an occluder edge / through its centre / far from it;
              an occluder at the segment's end
The candidate sets are pinned by closed-form cases and, on real scenes, by brute force: the
nearest hit of every ray turned by up to the band around an ID-fragile primary ray must be one of
that pixel's candidates (soundness), and an ID-robust pixel's only candidate is its own hit.
"""
import math

import numpy as np

from oracle.oracle import (DEFAULT_EPS, FRAG_BOUNDARY, FRAG_COMPETE, FRAG_GRAZE, FRAG_RANGE, FRAG_SHADE,
                           FRAG_SHADOW, ID_FRAGILE_MASK, Oracle)
from paper_1702_01530_b200 import scenes
from paper_1702_01530_b200.scenes import material
from tests.test_oracle_pins import mk_scene

EPS_T = 1e-4
EPS_E = DEFAULT_EPS["eps_edge"]      # the triangle-edge band (angular)
T_MIN = 1e-4
BIG = 50.0


def quad(z, lo=-BIG, hi=BIG, x0=None):
    """Two triangles covering [lo,hi]^2 (or [x0,hi] x [lo,hi]) in the plane z, CCW from -z."""
    xa = lo if x0 is None else x0
    return [[xa, lo, z], [hi, lo, z], [xa, hi, z], [hi, hi, z]], [[0, 1, 2], [1, 3, 2]]


def stacked(dz):
    """Triangle A (ID 0) at z = 5 and triangle B (ID 1) at z = 5 + dz, both large."""
    v = [[-BIG, -BIG, 5.0], [BIG, -BIG, 5.0], [0.0, BIG, 5.0],
         [-BIG, -BIG, 5.0 + dz], [BIG, -BIG, 5.0 + dz], [0.0, BIG, 5.0 + dz]]
    return Oracle(mk_scene(verts=v, tris=[[0, 1, 2], [3, 4, 5]]))


O = np.zeros(3)
DZ = np.array([0.0, 0.0, 1.0])


def test_f1_compete_stacked_triangles():
    """F1: another primitive hit within eps_t * t* of the nearest hit (t* = 5)."""
    for dz, want in ((0.0, True), (0.5 * EPS_T * 5, True), (-0.5 * EPS_T * 5, True),
                     (2.0 * EPS_T * 5, False), (-2.0 * EPS_T * 5, False)):
        o = stacked(dz)
        f, _ = o.ray_flags(O, DZ)
        assert bool(f & FRAG_COMPETE) == want, (dz, f)
        assert not f & (FRAG_GRAZE | FRAG_RANGE | FRAG_BOUNDARY), (dz, f)
        cand, _ = o.ray_candidates(O, DZ)
        assert cand == ([0, 1] if want else [0 if dz > 0 else 1]), (dz, cand)


def test_f4_grazing():
    """F4: |n.d| <= eps_t at the hit.  Plane y = 0 (no boundary), ray from (0, 1, 0) descending at
    |n.d| = a: hit at t = 1/a."""
    o = Oracle(mk_scene(planes=[[0, 1, 0, 0]]))
    for a, want in ((5e-5, True), (2e-4, False), (1e-3, False)):
        d = np.array([math.sqrt(1 - a * a), -a, 0.0])
        t, pid = o.nearest([0, 1, 0], d)
        assert pid == 0 and abs(t - 1 / a) <= 1e-9 / a
        f, _ = o.ray_flags([0, 1, 0], d)
        assert f == (FRAG_GRAZE if want else 0), (a, f)
        cand, _ = o.ray_candidates([0, 1, 0], d)
        assert cand == ([-1, 0] if want else [0]), (a, cand)    # a grazing plane is never robust


def test_f5_range_near_t_min():
    """F5: a candidate t within eps_abs (1 + |o|_inf) = 1e-5 of t_min = 1e-4 (origin at 0)."""
    for z, flag, hit in ((T_MIN + 5e-6, True, True), (T_MIN - 5e-6, True, False),
                         (T_MIN + 5e-5, False, True), (T_MIN - 5e-5, False, False)):
        v, t = quad(z)
        o = Oracle(mk_scene(verts=v, tris=t))
        _, pid = o.nearest(O, DZ)
        assert (pid >= 0) == hit, (z, pid)
        f, _ = o.ray_flags(O, DZ)
        assert bool(f & FRAG_RANGE) == flag, (z, f)
        cand, _ = o.ray_candidates([0.25, 0.1, 0], DZ)          # off the quad's diagonal edge
        if flag:
            assert -1 in cand and (0 in cand or 1 in cand), (z, cand)
        else:
            assert cand == ([1] if hit else [-1]), (z, cand)           # (0.25, 0.1): x + y > 0 -> tri 1


def _plane_hit_with_light(ndl):
    """Primary ray straight down onto the diffuse plane y = 0 at the origin; one light at unit
    distance whose direction makes n.l = ndl with the plane normal."""
    light = [math.sqrt(1 - ndl * ndl), ndl, 0.0, 1.0, 1.0, 1.0]
    return Oracle(mk_scene(planes=[[0, 1, 0, 0]], mats=[material(0.5, 0.3, 8)], lights=[light]))


def test_f6_shading_gate():
    """F6 (reading 2 gate): |n.l| <= eps_t flags the pixel; the light's term is on only for n.l > 0."""
    for ndl, want in ((5e-5, True), (-5e-5, True), (2e-4, False), (-2e-4, False), (0.5, False)):
        o = _plane_hit_with_light(ndl)
        rgb, cnt, fl = o.trace_ray_ex([0, 1, 0], [0, -1, 0], 0)
        assert bool(fl & FRAG_SHADE) == want, (ndl, fl)
        assert cnt[3] == (1 if ndl > 0 else 0)                    # a shadow ray only past the gate
        assert (rgb[0] > 0) == (ndl > 0)


def test_f6_tir_switch():
    """F6 (reading 5): the TIR discriminant k = 1 - eta^2 (1 - cos_i^2) within eps_t of 0.  A ray
    leaving a glass half-space (plane y = 0, ior 1.5, seen from its back side: eta = ior) at
    cos_i chosen for a given k."""
    ior = 1.5
    glass = material(0.0, 0.0, 1.0, kr=0.0, kt=1.0, ior=ior)
    for k, want in ((5e-5, True), (-5e-5, True), (1e-2, False), (-1e-2, False)):
        cos_i = math.sqrt(1 - (1 - k) / ior ** 2)
        d = np.array([math.sqrt(1 - cos_i ** 2), cos_i, 0.0])        # upward, hits y = 0 from below
        o = Oracle(mk_scene(planes=[[0, 1, 0, 0]], mats=[glass], background=0.5))
        _, cnt, fl = o.trace_ray_ex([0, -1, 0], d, 1)
        assert bool(fl & FRAG_SHADE) == want, (k, fl)
        assert cnt[1] == (1 if k < 0 else 0) and cnt[2] == (1 if k >= 0 else 0), (k, cnt)   # TIR -> reflection


def test_shadow_flags():
    """Shadow query over (t_min, dist = 10) along +z from the origin; occluder triangle in z = 5.
    Fragile (SHADOW) only when no primitive robustly blocks the segment and a boundary passes
    within eps_edge * t of it, or a candidate t sits at the segment's end."""
    def occ(x0):
        v, t = quad(5.0, x0=x0)
        return Oracle(mk_scene(verts=v, tris=t))
    t_edge = 5.0
    for x0, want in ((0.5 * EPS_E * t_edge, True),     # misses the occluder, 0.5 eps_edge t from its edge
                     (-0.5 * EPS_E * t_edge, True),    # blocked, but only 0.5 eps_edge t inside the edge
                     (3.0 * EPS_E * t_edge, False),    # misses it by 3 eps_edge t: robust
                     (-1.0, False),                # through the occluder's interior: robust
                     (2e-4 * t_edge, False)):      # misses by 2e-4 t: robustly unoccluded
        f, _ = occ(x0).ray_flags(O, DZ, kind="shadow", dist=10.0)
        assert f == (FRAG_SHADOW if want else 0), (x0, f)
    # an occluder at the segment's end (the light sits on a surface): fragile
    for z, want in ((10.0 * (1 - 0.5e-4), True), (10.0 * (1 + 0.5e-4), True), (10.0 * (1 + 3e-4), False)):
        v, t = quad(z)
        f, _ = Oracle(mk_scene(verts=v, tris=t)).ray_flags([0.3, 0.1, 0], DZ, kind="shadow", dist=10.0)
        assert f == (FRAG_SHADOW if want else 0), (z, f)


def test_candidates_closed_form():
    """Near-tie candidates (reading 22): the IDs a band-turned ray may hit first."""
    # robust interior hit of one triangle of a quad: only that triangle
    v, t = quad(5.0, lo=-1, hi=1)
    o = Oracle(mk_scene(verts=v, tris=t))
    assert o.ray_candidates([-0.5, -0.5, 0], DZ)[0] == [0]
    assert o.ray_candidates([0.5, 0.5, 0], DZ)[0] == [1]
    # on the shared diagonal edge (1,-1)-(-1,1): both -- and a miss, because neither triangle is
    # hit robustly and FP32 Moller-Trumbore is not watertight across a shared edge
    assert o.ray_candidates(O, DZ)[0] == [-1, 0, 1]
    # 0.5 eps_edge * t off the diagonal (distance measured in the plane): still all; 3x: one
    for off, want in ((0.5 * EPS_E * 5, [-1, 0, 1]), (3 * EPS_E * 5, [1])):
        p = np.array([1.0, 1.0, 0.0]) / math.sqrt(2) * off
        assert o.ray_candidates(p, DZ)[0] == want, off
    # the quad's outer edge at x = 1: inside by 0.5 band -> {tri, miss}; outside by 0.5 band too
    for x, want in ((1 - 0.5 * EPS_E * 5, [-1, 1]), (1 + 0.5 * EPS_E * 5, [-1, 1]), (1 + 3 * EPS_E * 5, [-1])):
        assert o.ray_candidates([x, 0.5, 0], DZ)[0] == want, x
    # sphere silhouette (centre (1,0,10), r = 1, ray along x = 0): sphere or miss; with a plane
    # behind it: sphere or plane (a robust hit exists, so no miss)
    s = Oracle(mk_scene(spheres=[[1.0, 0, 10, 1.0]]))
    assert s.ray_candidates(O, DZ)[0] == [-1, 0]
    s = Oracle(mk_scene(spheres=[[1.0, 0, 10, 1.0]], planes=[[0, 0, 1, 20]]))
    assert s.ray_candidates(O, DZ)[0] == [0, 1]
    # ... and 2e-4 relative inside the silhouette: the sphere robustly
    s = Oracle(mk_scene(spheres=[[1.0 - 2e-4 * 10, 0, 10, 1.0]], planes=[[0, 0, 1, 20]]))
    assert s.ray_candidates(O, DZ)[0] == [0]
    # a triangle in front whose edge the ray grazes: it or the robust quad behind it; clear of the
    # edge, only the quad (tri 2 at z = 4 with its hypotenuse on x + y = 0.2)
    v2 = v + [[-1, -1, 4.0], [1.2, -1, 4.0], [-1, 1.2, 4.0]]
    o = Oracle(mk_scene(verts=v2, tris=t + [[4, 5, 6]]))
    assert o.ray_candidates([0.1, 0.1, 0], DZ)[0] == [1, 2]
    assert o.ray_candidates([0.5, 0.5, 0], DZ)[0] == [1]
    assert o.ray_candidates([-0.5, -0.5, 0], DZ)[0] == [2]      # robustly inside tri 2: the quad is behind


def _perturbed(d, alpha, rng, n):
    a = np.array([0.0, 1, 0]) if abs(d[1]) < 0.9 else np.array([1.0, 0, 0])
    u = np.cross(d, a)
    u /= np.linalg.norm(u)
    w = np.cross(d, u)
    out = []
    for _ in range(n):
        phi = rng.uniform(0, 2 * math.pi)
        r = alpha * math.sqrt(rng.uniform(0, 1))
        q = d + r * (math.cos(phi) * u + math.sin(phi) * w)
        out.append(q / np.linalg.norm(q))
    return out


def _tangent_dir(eye, c, r, rng):
    """A unit direction from eye grazing the sphere (c, r): its silhouette."""
    w = c - eye
    L = np.linalg.norm(w)
    w /= L
    a = np.array([0.0, 1, 0]) if abs(w[1]) < 0.9 else np.array([1.0, 0, 0])
    u = np.cross(w, a)
    u /= np.linalg.norm(u)
    v = np.cross(w, u)
    phi = rng.uniform(0, 2 * math.pi)
    axis = math.cos(phi) * u + math.sin(phi) * v
    al = math.asin(r / L)
    return math.cos(al) * w + math.sin(al) * axis


def test_candidates_sound_under_perturbation():
    """Soundness by brute force.  Rays from the C3 eye aimed at points ON mesh edges and vertices
    and tangent to sphere silhouettes: the ray's own nearest hit is a candidate, and so is the
    nearest hit of every ray turned by up to 0.9 x eps_edge (the triangle band; sphere bands are
    wider).  ID-robust pixels of a small render have exactly their hit as the only candidate (two
    independent code paths of the oracle agree)."""
    rng = np.random.default_rng(11)
    sc = scenes.scene_c3()
    o = Oracle(sc)
    cam = o.camera()
    eye = np.asarray(cam.eye[0][:], np.float64)
    rays = []
    for k in range(40):
        tri = sc.tris[rng.integers(len(sc.tris))]
        a, b = sc.vertices[tri[k % 3]], sc.vertices[tri[(k + 1) % 3]]
        p = a + (0.0 if k % 8 == 0 else rng.uniform(0, 1)) * (b - a)      # every 8th: a vertex
        d = p - eye
        rays.append(d / np.linalg.norm(d))
    for k in range(20):
        c = sc.spheres[rng.integers(len(sc.spheres))]
        rays.append(_tangent_dir(eye, c[:3], c[3], rng))
    sizes = []
    for d in rays:
        cand, n = o.ray_candidates(eye, d)
        assert n == len(cand) and n <= 8, (n, cand)
        assert o.nearest(eye, d)[1] in cand, cand
        for dq in _perturbed(d, 0.9 * EPS_E, rng, 24):
            assert o.nearest(eye, dq)[1] in cand, cand
        sizes.append(n)
    assert max(sizes) >= 2                                  # the cases are near ties indeed
    s = sc.with_view(width=48, height=27)
    out = o.render(rig=s.rig, width=48, height=27)
    robust = np.argwhere((out["pflags"] & ID_FRAGILE_MASK) == 0)
    for e, py, px in robust[rng.choice(len(robust), 40, replace=False)]:
        org, d = o.primary_ray(o.camera(width=48, height=27), int(e), int(px), int(py))
        assert o.ray_candidates(org, d)[0] == [int(out["id"][e, py, px])], (e, py, px)
    frag = np.argwhere((out["pflags"] & ID_FRAGILE_MASK) != 0)
    for e, py, px in frag:
        n = int(out["ncand"][e, py, px])
        assert n >= 1 and int(out["id"][e, py, px]) in out["cand"][e, py, px][:n]
