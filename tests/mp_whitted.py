"""High-precision (mpmath) evaluation of the stereo Whitted definition, one pixel at a time.
TEST INFRASTRUCTURE ONLY: the "double-precision adequacy" pin of SURVEY.md §8(c) -- the oracle
(double, C) must agree with this 40-digit evaluation to 1e-9 on non-fragile pixels.

Written from SURVEY.md §8(c) steps 1-5 (and the DESIGN.md readings it cites), independently of
oracle/whitted_oracle.c: different language, different arithmetic, and a different triangle
formulation (explicit 3x3 Cramer solve of o + t d = v0 + u e1 + v e2 instead of Moller-Trumbore;
the two are the same function of exact inputs).  Slow: use on a handful of pixels.
"""
from __future__ import annotations

import mpmath as mp

mp.mp.dps = 40
T_MIN = mp.mpf("1e-4")       # S:156, R#8
BIAS = mp.mpf("1e-4")        # S:193, R#8


def V(a):
    return [mp.mpf(float(x)) for x in a]


def add(a, b):
    return [a[0] + b[0], a[1] + b[1], a[2] + b[2]]


def sub(a, b):
    return [a[0] - b[0], a[1] - b[1], a[2] - b[2]]


def scl(a, s):
    return [a[0] * s, a[1] * s, a[2] * s]


def dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def cross(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def norm(a):
    return scl(a, 1 / mp.sqrt(dot(a, a)))


def det3(c0, c1, c2):
    """det of the 3x3 matrix with columns c0, c1, c2."""
    return dot(c0, cross(c1, c2))


class MpScene:
    def __init__(self, scene):
        self.spheres = [(V(s[:3]), mp.mpf(float(s[3]))) for s in scene.spheres]
        self.planes = [(V(p[:3]), mp.mpf(float(p[3]))) for p in scene.planes]
        vt = [V(v) for v in scene.vertices]
        self.tris = [(vt[int(a)], vt[int(b)], vt[int(c)]) for a, b, c in scene.tris]
        self.smat = [int(m) for m in scene.sphere_mat]
        self.pmat = [int(m) for m in scene.plane_mat]
        self.tmat = [int(m) for m in scene.tri_mat]
        self.mats = [[mp.mpf(float(x)) for x in m] for m in scene.materials]
        self.lights = [(V(l[:3]), V(l[3:6])) for l in scene.lights]
        self.ambient = V(scene.ambient)
        self.background = V(scene.background)

    # ---- step 3: candidates with t > t_min; (t, global id) lexicographic minimum
    def hits(self, o, d):
        """All strict hits (t, gid, kind, index) along the ray."""
        out = []
        S, P = len(self.spheres), len(self.planes)
        for i, (c, r) in enumerate(self.spheres):
            oc = sub(o, c)
            b = dot(oc, d)
            c0 = dot(oc, oc) - r * r
            disc = b * b - c0
            if disc < 0:
                continue
            sq = mp.sqrt(disc)
            for t in (-b - sq, -b + sq):
                if t > T_MIN:
                    out.append((t, i, "s", i))
                    break
        for i, (n, k) in enumerate(self.planes):
            nd = dot(n, d)
            if nd == 0:
                continue
            t = (k - dot(n, o)) / nd
            if t > T_MIN:
                out.append((t, S + i, "p", i))
        for i, (v0, v1, v2) in enumerate(self.tris):
            e1, e2 = sub(v1, v0), sub(v2, v0)
            # o + t d = v0 + u e1 + v e2  <=>  [-d e1 e2] (t u v)^T = o - v0   (Cramer)
            nd = scl(d, -1)
            rhs = sub(o, v0)
            D = det3(nd, e1, e2)
            if D == 0:
                continue
            t = det3(rhs, e1, e2) / D
            u = det3(nd, rhs, e2) / D
            v = det3(nd, e1, rhs) / D
            if u >= 0 and v >= 0 and u + v <= 1 and t > T_MIN:
                out.append((t, S + P + i, "t", i))
        return out

    def nearest(self, o, d):
        h = self.hits(o, d)
        return min(h, key=lambda x: (x[0], x[1])) if h else None

    def occluded(self, o, d, dist):
        return any(t < dist for t, _, _, _ in self.hits(o, d))

    # ---- step 4: Trace(ray, depth)
    def trace(self, o, d, depth):
        h = self.nearest(o, d)
        if h is None:
            return list(self.background)
        t, gid, kind, i = h
        p = add(o, scl(d, t))
        if kind == "s":
            c, r = self.spheres[i]
            ng = scl(sub(p, c), 1 / r)
            m = self.mats[self.smat[i]]
        elif kind == "p":
            ng = norm(self.planes[i][0])
            m = self.mats[self.pmat[i]]
        else:
            v0, v1, v2 = self.tris[i]
            ng = norm(cross(sub(v1, v0), sub(v2, v0)))
            m = self.mats[self.tmat[i]]
        kd, ks, shin, kr, kt, ior = m[0:3], m[3:6], m[6], m[7], m[8], m[9]
        front = dot(d, ng) < 0
        nf = ng if front else scl(ng, -1)
        col = [self.ambient[k] * kd[k] for k in range(3)]
        for Lp, I in self.lights:
            l = norm(sub(Lp, p))
            ndl = dot(nf, l)
            if ndl <= 0:                                                    # R#2 gate
                continue
            os_ = add(p, scl(nf, BIAS))
            sv = sub(Lp, os_)
            dist = mp.sqrt(dot(sv, sv))
            if self.occluded(os_, scl(sv, 1 / dist), dist):               # R#3, R#4
                continue
            rv = sub(scl(nf, 2 * ndl), l)
            rdv = -dot(rv, d)
            spec = rdv ** shin if rdv > 0 else mp.mpf(0)
            for k in range(3):
                col[k] += kd[k] * I[k] * ndl + ks[k] * I[k] * spec
        if depth > 0:
            kr_eff = kr
            if kt > 0:
                eta = 1 / ior if front else ior
                cosi = -dot(d, nf)
                kk = 1 - eta * eta * (1 - cosi * cosi)
                if kk < 0:
                    kr_eff += kt                                            # R#5 TIR
                else:
                    td = norm(add(scl(d, eta), scl(nf, eta * cosi - mp.sqrt(kk))))
                    tc = self.trace(sub(p, scl(nf, BIAS)), td, depth - 1)
                    col = [col[k] + kt * tc[k] for k in range(3)]
            if kr_eff > 0:
                rd = norm(sub(d, scl(nf, 2 * dot(d, nf))))
                rc = self.trace(add(p, scl(nf, BIAS)), rd, depth - 1)
                col = [col[k] + kr_eff * rc[k] for k in range(3)]
        return col


def primary_ray(rig, W, H, eye, px, py):
    """Steps 1-2: rig basis, eye positions, off-axis shift, pixel-centre ray (R#13)."""
    e, la, up = V(rig.eye), V(rig.look_at), V(rig.up)
    f = norm(sub(la, e))
    r = norm(cross(f, up))
    u = cross(r, f)
    s = mp.mpf(float(rig.interocular))
    C = float(rig.convergence)
    eye_pos = sub(e, scl(r, s / 2)) if eye == 0 else add(e, scl(r, s / 2))
    sigma = mp.mpf(0)
    if C > 0 and C != float("inf"):
        sigma = (s / (2 * mp.mpf(C))) * (1 if eye == 0 else -1)
    th = mp.tan(mp.radians(mp.mpf(float(rig.vfov_deg))) / 2)
    a = mp.mpf(W) / H
    sx = (2 * (mp.mpf(px) + mp.mpf("0.5")) / W - 1) * th * a
    sy = (1 - 2 * (mp.mpf(py) + mp.mpf("0.5")) / H) * th
    d = norm(add(add(f, scl(r, sx + sigma)), scl(u, sy)))
    return eye_pos, d


def render_pixel(scene, eye, px, py, width=None, height=None, max_depth=None):
    W = width or scene.width
    H = height or scene.height
    D = scene.max_depth if max_depth is None else max_depth
    ms = MpScene(scene)
    o, d = primary_ray(scene.rig, W, H, eye, px, py)
    return [float(x) for x in ms.trace(o, d, D)]
