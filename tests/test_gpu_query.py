"""GPU ray queries through the C ABI (rt_intersect: the renderer's own nearest-hit / any-hit device
code on caller rays):
  - the device intersectors against closed forms (SURVEY §8(c) pins: ray-sphere, ray-plane, the
    SPEC.md:176-178 triangle examples, S:187 stacked triangles, S:300 shared-edge tie);
  - BVH traversal == brute force, bit for bit (t and ID; occlusion flags), on 2^17 seeded random
    rays per scene from inside and around the scene bounds -- rays the camera never shoots;
  - GPU vs the double-precision oracle on random rays: IDs equal off the oracle's fragile set
    (reading 22, F1-F5), t within FP32 rounding.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import ID_FRAGILE_MASK, Oracle  # noqa: E402
from paper_1702_01530_b200 import rt, scenes  # noqa: E402
from paper_1702_01530_b200.scenes import Scene  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = rt.StereoRenderer(0)
    yield r
    r.close()


def _dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float32), device="cuda")


def nearest(R, o, d, brute=False):
    t, i = rt.rt_intersect(R.ctx, _dev(o), _dev(d), brute=brute)
    torch.cuda.synchronize()
    return t.cpu().numpy(), i.cpu().numpy()


def occluded(R, o, d, tmax, brute=False):
    f = rt.rt_intersect(R.ctx, _dev(o), _dev(d), _dev(tmax), any_hit=True, brute=brute)
    torch.cuda.synchronize()
    return f.cpu().numpy()


def _base(name):
    s = Scene(name)
    s.materials = np.stack([scenes.material(0.5, 0.2, 8.0)])
    s.lights = np.array([[0.0, 10.0, 0.0, 1.0, 1.0, 1.0]])
    s.ambient = np.full(3, 0.1)
    s.background = np.zeros(3)
    s.rig = scenes._rig((0.0, 0.0, 10.0), (0.0, 0.0, 0.0), 40.0)
    s.width, s.height, s.max_depth = 8, 8, 1
    return s


def test_sphere_closed_form(R):
    """Ray (h, 0, 0) + t (0, 0, -1) vs the sphere c = (0, 0, -10), r = 2: t = 10 - sqrt(4 - h^2)
    for |h| < 2, a miss beyond; from the centre, t = r (SURVEY §8(c) pins)."""
    s = _base("sphere")
    s.spheres = np.array([[0.0, 0.0, -10.0, 2.0]])
    s.sphere_mat = np.zeros(1, np.uint32)
    R.upload(s.finalize())
    h = np.array([-1.9, -1.5, -1.0, -0.5, 0.0, 0.25, 0.75, 1.25, 1.75, 1.95, 2.05, 3.0])
    o = np.stack([h, np.zeros_like(h), np.zeros_like(h)], 1)
    d = np.tile([0.0, 0.0, -1.0], (len(h), 1))
    t, i = nearest(R, o, d)
    inside = np.abs(h) < 2
    np.testing.assert_allclose(t[inside], 10.0 - np.sqrt(4.0 - h[inside] ** 2), rtol=2e-6)
    assert np.all(i[inside] == 0) and np.all(i[~inside] == -1) and np.all(np.isinf(t[~inside]))
    t, i = nearest(R, [[0.0, 0.0, -10.0]], [[0.3, -0.4, 0.5]])
    assert i[0] == 0 and abs(t[0] - 2.0) <= 2e-6


def test_plane_closed_form(R):
    """Ray (0, 2, 0), d = (1, -1, 0)/sqrt 2 vs the plane y = 0: t = 2 sqrt 2; parallel -> miss."""
    s = _base("plane")
    s.planes = np.array([[0.0, 1.0, 0.0, 0.0]])
    s.plane_mat = np.zeros(1, np.uint32)
    R.upload(s.finalize())
    t, i = nearest(R, [[0.0, 2.0, 0.0], [0.0, 2.0, 0.0]], [[1.0, -1.0, 0.0], [1.0, 0.0, 0.0]])
    assert i[0] == 0 and abs(t[0] - 2 * math.sqrt(2)) <= 4e-6
    assert i[1] == -1 and np.isinf(t[1])


def test_triangle_spec_examples(R):
    """triangle (-1,-1,5) (3,-1,5) (-1,3,5); a ray along +z from the origin hits at
    t = 5, along -z misses, in the triangle's plane misses.  S:187 stacked triangles at z = 5 and 7
    -> 5.  S:300 a ray through the shared edge of two triangles -> the smaller ID."""
    s = _base("tri")
    s.vertices = np.array([[-1, -1, 5], [3, -1, 5], [-1, 3, 5], [-1, -1, 7], [3, -1, 7], [-1, 3, 7]], float)
    s.tris = np.array([[3, 4, 5], [0, 1, 2]], np.uint32)          # the far triangle gets the smaller ID
    s.tri_mat = np.zeros(2, np.uint32)
    R.upload(s.finalize())
    t, i = nearest(R, [[0, 0, 0], [0, 0, 0], [-5, 0, 5]], [[0, 0, 1], [0, 0, -1], [1, 0, 0]])
    assert i[0] == 1 and abs(t[0] - 5.0) <= 1e-5
    assert i[1] == -1 and i[2] == -1
    f = occluded(R, [[0, 0, 0], [0, 0, 0]], [[0, 0, 1], [0, 0, 1]], [6.0, 4.0])
    assert f.tolist() == [1, 0]                                    # strict t < tmax
    # shared edge: two triangles of the unit quad at z = 5, ray through the diagonal
    q = _base("quad")
    q.vertices = np.array([[0, 0, 5], [1, 0, 5], [1, 1, 5], [0, 1, 5]], float)
    q.tris = np.array([[0, 2, 3], [0, 1, 2]], np.uint32)
    q.tri_mat = np.zeros(2, np.uint32)
    R.upload(q.finalize())
    t, i = nearest(R, [[0.5, 0.5, 0.0]], [[0, 0, 1]])
    assert i[0] == 0 and abs(t[0] - 5.0) <= 1e-5


def _random_rays(s, n, seed):
    """Origins uniform in the scene's bounds grown by 50 % (so about 1/3 start inside), directions
    uniform on the sphere, any-hit lengths uniform in (0, 2 x diagonal]."""
    pts = [s.vertices.reshape(-1, 3)] if s.n_tris else []
    if s.n_spheres:
        pts += [s.spheres[:, :3] - s.spheres[:, 3:], s.spheres[:, :3] + s.spheres[:, 3:]]
    pts = np.concatenate(pts)
    lo, hi = pts.min(0), pts.max(0)
    c, e = (lo + hi) / 2, (hi - lo) * 0.75
    rng = np.random.Generator(np.random.PCG64(seed))
    o = c + rng.uniform(-1, 1, (n, 3)) * e
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tmax = rng.uniform(1e-3, 1, n) * 2 * np.linalg.norm(hi - lo)
    return o, d, tmax


@pytest.mark.parametrize("name", ["C2", "C3", "paper6", "urchin"])
def test_random_rays_bvh_equals_bruteforce(R, name):
    s = scenes.paper_scene(6) if name == "paper6" else scenes.scene_urchin() if name == "urchin" else scenes.make_scene(name)
    R.upload(s)
    o, d, tmax = _random_rays(s, 1 << 17, 21)
    t1, i1 = nearest(R, o, d)
    t2, i2 = nearest(R, o, d, brute=True)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(t1.view(np.uint32), t2.view(np.uint32))
    assert 0.05 < (i1 >= 0).mean() < 0.999                        # the rays exercise hits and misses
    f1 = occluded(R, o, d, tmax)
    f2 = occluded(R, o, d, tmax, brute=True)
    np.testing.assert_array_equal(f1, f2)
    assert 0.02 < f1.mean() < 0.98


def test_random_rays_bvh_equals_bruteforce_1m_triangles(R):
    """The bench scene (C4, 1M triangles): 8 192 random rays, BVH == brute force bit for bit."""
    s = scenes.scene_c4()
    R.upload(s)
    o, d, tmax = _random_rays(s, 8192, 22)
    t1, i1 = nearest(R, o, d)
    t2, i2 = nearest(R, o, d, brute=True)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(t1.view(np.uint32), t2.view(np.uint32))
    np.testing.assert_array_equal(occluded(R, o, d, tmax), occluded(R, o, d, tmax, brute=True))


def test_random_rays_vs_oracle(R):
    """C3 (triangles and spheres): GPU nearest hits of 2 048 random rays vs the oracle's double
    brute force: IDs equal wherever the oracle's F1-F5 flags leave the decision robust, t within
    FP32 rounding of the hit distance; occlusion equal where the shadow query is robust."""
    s = scenes.scene_c3()
    R.upload(s)
    o, d, tmax = _random_rays(s, 2048, 23)
    # half of the rays aimed at a random vertex (jittered), so most of them hit something
    rng = np.random.Generator(np.random.PCG64(24))
    v = s.vertices[rng.integers(0, len(s.vertices), len(o) // 2)] + rng.normal(scale=0.05, size=(len(o) // 2, 3))
    a = v - o[: len(o) // 2]
    d[: len(o) // 2] = a / np.linalg.norm(a, axis=1, keepdims=True)
    o32, d32 = o.astype(np.float32), d.astype(np.float32)
    t, i = nearest(R, o32, d32)
    f = occluded(R, o32, d32, tmax.astype(np.float32))
    O = Oracle(s)
    robust = ok_t = n_hit = 0
    for k in range(len(o)):
        ok = o32[k].astype(np.float64)
        dk = d32[k].astype(np.float64)
        dk = dk / np.linalg.norm(dk)
        tr, ir = O.nearest(ok, dk)
        fl, _ = O.ray_flags(ok, dk)
        if fl & ID_FRAGILE_MASK:
            continue
        robust += 1
        assert i[k] == ir, (k, i[k], ir, fl)
        if ir >= 0:
            n_hit += 1
            assert abs(t[k] - tr) <= 1e-5 * (tr + np.abs(ok).max()), (k, t[k], tr)
            ok_t += 1
        sf, _ = O.ray_flags(ok, dk, "shadow", float(np.float32(tmax[k])))
        if not sf:
            occ = math.isfinite(tr) and 1e-4 < tr < float(np.float32(tmax[k]))
            assert f[k] == int(occ), (k, f[k], tr, tmax[k])
    assert robust > 0.95 * len(o) and n_hit > 600
