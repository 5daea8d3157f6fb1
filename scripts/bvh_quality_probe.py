"""BVH quality probe: build time, BVH4 node visits and primitive tests per ray, and stereo-frame
time (median of 10, 4 frames in flight excluded) for the configs given.  Run it twice to compare
builds, e.g. with RT_HOST_SAH=1 (host binned-SAH BVH2 in place of the LBVH + treelets, an
experiment).  usage: python scripts/bvh_quality_probe.py [C3 C4 ...] > out.json
"""
import json
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from kd_ablation import counts, frame_ms  # noqa: E402
from paper_1702_01530_b200 import rt, scenes  # noqa: E402


def main():
    names = sys.argv[1:] or ["C3", "C4"]
    R = rt.StereoRenderer(0)
    res = {"RT_HOST_SAH": os.environ.get("RT_HOST_SAH", "0")}
    for name in names:
        s = scenes.make_scene(name)
        info = R.upload(s)
        R.set_camera(s.rig)
        fb = R.alloc_fb(s.width, s.height)
        c, rays, ids = counts(R, s)
        ms = frame_ms(R, s, fb)
        res[name] = {"build_ms": info["build_us"] / 1e3, "bvh_nodes": info["bvh_nodes"], "bvh_depth": info["bvh_depth"],
                     "ms": ms, "mrays_s": rays / ms / 1e3, "node_visits_per_ray": c["node_visits"] / rays,
                     "prim_tests_per_ray": (c["tri_tests"] + c["sphere_tests"]) / rays}
        print(name, res[name], file=sys.stderr, flush=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
