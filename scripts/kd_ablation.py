"""NEXT-4 ablation (Table 1): the device LBVH4 (product path)
against a binned-SAH kd-tree over the same primitive records and FP32 intersectors, on the
BASELINE configs.  Per structure: build time, device bytes, depth, stereo-frame time (median of
10, events on the render stream), node visits and primitive tests per ray, and whether the
primary hit IDs equal the BVH's.  usage: python scripts/kd_ablation.py [C2 C3 C4 ...] > out.json
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

KD_CONFIGS = [(1, 0), (2, 0), (4, 0), (8, 0), (1, 24)]


def frame_ms(R, s, fb, **kw):
    for _ in range(3):
        R.render(s.width, s.height, s.max_depth, fb=fb, **kw)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(10):
        ev[0].record()
        R.render(s.width, s.height, s.max_depth, fb=fb, **kw)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return float(np.median(ts))


def counts(R, s, **kw):
    out = R.render(s.width, s.height, s.max_depth, count=True, want_id=True, **kw)
    torch.cuda.synchronize()
    c = R.counters_dict(out["counters"])
    rays = c["primary"] + c["reflection"] + c["refraction"] + c["shadow"]
    return c, rays, out["id"].cpu().numpy()


def main():
    names = sys.argv[1:] or ["C2", "C3", "C4"]
    R = rt.StereoRenderer(0)
    res = {}
    for name in names:
        s = scenes.make_scene(name)
        info = R.upload(s)
        R.set_camera(s.rig)
        fb = R.alloc_fb(s.width, s.height)
        c, rays, ids = counts(R, s)
        ms = frame_ms(R, s, fb)
        rows = [{"structure": "LBVH4 (device build, product)", "build_ms": info["build_us"] / 1e3,
                 "device_mb": info["device_bytes"] / 1e6, "depth": info["bvh_depth"], "nodes": info["bvh_nodes"],
                 "ms": ms, "mrays_s": rays / ms / 1e3, "node_visits_per_ray": c["node_visits"] / rays,
                 "prim_tests_per_ray": (c["tri_tests"] + c["sphere_tests"]) / rays, "ids_equal_bvh": True}]
        for ml, md in KD_CONFIGS:
            t0 = time.time()
            k = rt.rt_kdtree_build(R.ctx, ml, md)
            wall = time.time() - t0
            kc, krays, kids = counts(R, s, kdtree=True)
            kms = frame_ms(R, s, fb, kdtree=True)
            rows.append({"structure": f"kd-tree SAH (host build) max_leaf {ml} max_depth {md or 'auto'}",
                         "build_ms": k["kd_build_us"] / 1e3, "build_wall_s": wall,
                         "device_mb": k["kd_device_bytes"] / 1e6, "depth": k["kd_depth"], "nodes": k["kd_nodes"],
                         "refs_per_prim": k["kd_refs"] / max(info["bvh_prims"], 1), "leaves": k["kd_leaves"],
                         "ms": kms, "mrays_s": krays / kms / 1e3, "node_visits_per_ray": kc["node_visits"] / krays,
                         "prim_tests_per_ray": (kc["tri_tests"] + kc["sphere_tests"]) / krays,
                         "ids_equal_bvh": bool(np.array_equal(kids, ids)), "rays_equal_bvh": krays == rays})
            print(name, rows[-1], file=sys.stderr, flush=True)
        res[name] = {"workload": f"{name}: {s.width}x{s.height} per eye, {s.n_tris} tris + {s.n_spheres} spheres, "
                                 f"depth {s.max_depth}", "rays_per_frame": rays, "rows": rows}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
