"""Scene upload + device BVH build time of a config (rt_scene_info build_us), a few repeats.

    python scripts/build_time.py [C4] [repeats]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s = scenes.make_scene(name)
R = rt.StereoRenderer(0)
for k in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    R.upload(s)
    torch.cuda.synchronize()
    info = rt.rt_scene_info(R.ctx)
    print(f"{name} upload {1e3 * (time.perf_counter() - t0):.1f} ms, build {info['build_us'] / 1e3:.1f} ms "
          f"(incl. host validation), nodes {info['bvh_nodes']}, depth {info['bvh_depth']}", flush=True)
