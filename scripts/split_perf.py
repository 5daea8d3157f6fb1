"""Cost split of the C4 frame by ray kind (development aid)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402


def timeit(R, s, fb, n=10):
    for _ in range(3):
        R.render(s.width, s.height, s.max_depth, fb=fb)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(n):
        e[0].record()
        R.render(s.width, s.height, s.max_depth, fb=fb)
        e[1].record()
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]))
    return float(np.median(ts))


name = sys.argv[1] if len(sys.argv) > 1 else "C4"
base = scenes.make_scene(name)
R = rt.StereoRenderer(0)
fb = R.alloc_fb(base.width, base.height)
for label, depth, nl in [("full", base.max_depth, None), ("depth0", 0, None), ("primary only", 0, 0),
                         ("no shadows", base.max_depth, 0), ("1 light d0", 0, 1)]:
    s = base.with_view(max_depth=depth)
    if nl is not None:
        s.lights = base.lights[:nl]
    R.upload(s)
    R.set_camera(s.rig)
    out = R.render(s.width, s.height, s.max_depth, count=True)
    torch.cuda.synchronize()
    c = R.counters_dict(out["counters"])
    rays = c["primary"] + c["reflection"] + c["refraction"] + c["shadow"]
    ms = timeit(R, s, fb)
    print(f"{label:14s} {ms:7.3f} ms  rays {rays/1e6:6.2f}M  nodes/ray {c['node_visits']/rays:5.1f}  "
          f"tris/ray {c['tri_tests']/rays:5.2f}  {rays/ms/1e3:8.1f} Mrays/s", flush=True)
