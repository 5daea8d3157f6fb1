"""BVH build variants on the same scene (env knobs read at context creation): node visits per
ray, build time and the one-frame / in-flight render times.  usage: bvh_variants.py C4 [C3 ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

BASE = {"RT_SAH_SUBTREES": "2", "RT_TREELETS": "0"}
VARIANTS = [("fullSAH greedy collapse", {**BASE, "RT_COLLAPSE_DP": "0"})] + [
    (f"fullSAH DP collapse cprim={c}", {**BASE, "RT_COLLAPSE_DP": "1", "RT_COLLAPSE_CPRIM": c})
    for c in ("0.25", "0.4", "0.6", "1.0")]
if os.environ.get("RT_BVH_VARIANTS_OLD"):
    VARIANTS = [("subtrees16K+3treelets", {"RT_SAH_SUBTREES": "1", "RT_TREELETS": "3"}),
                ("fullSAH+0treelets", BASE)]


def time_frames(R, s, fb, flush, inflight=4, k=24):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for i in range(10):
        flush.zero_()
        ev[0].record()
        R.render(s.width, s.height, s.max_depth, fb=fb)
        ev[1].record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(ev[0].elapsed_time(ev[1]))
    streams = [torch.cuda.Stream() for _ in range(inflight)]
    fbs = [R.alloc_fb(s.width, s.height) for _ in range(inflight)]
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        st = torch.cuda.Event(enable_timing=True)
        st.record()
        for x in streams:
            x.wait_event(st)
        for j in range(k):
            x = streams[j % inflight]
            with torch.cuda.stream(x):
                flush.zero_()
            R.render(s.width, s.height, s.max_depth, fb=fbs[j % inflight], stream=x)
        ends = []
        for x in streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(x)
            ends.append(e)
        torch.cuda.synchronize()
        if rep:
            best = min(best, max(st.elapsed_time(e) for e in ends) / k)
    return float(np.median(ts)), best


def main():
    flush = torch.empty(160 * 2**20 // 4, dtype=torch.float32, device="cuda")
    out = {}
    for name in sys.argv[1:] or ["C4"]:
        s = scenes.make_scene(name)
        for label, env in VARIANTS:
            os.environ.update(env)
            R = rt.StereoRenderer(0)
            info = R.upload(s)
            R.set_camera(s.rig)
            c = R.counters_dict(R.render(s.width, s.height, s.max_depth, fb=False, count=True)["counters"])
            rays = c["primary"] + c["reflection"] + c["refraction"] + c["shadow"]
            fb = R.alloc_fb(s.width, s.height)
            one, pipe = time_frames(R, s, fb, flush)
            r = {"build_ms": info["build_us"] / 1e3, "bvh_nodes": info["bvh_nodes"], "depth": info["bvh_depth"],
                 "node_visits_per_ray": c["node_visits"] / rays, "box_tests_per_ray": c["box_tests"] / rays,
                 "tri_tests_per_ray": c["tri_tests"] / rays, "one_frame_ms": one, "inflight_ms": pipe}
            out[f"{name} {label}"] = r
            print(name, label, json.dumps(r), file=sys.stderr, flush=True)
            R.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
