"""Frame time / Mrays/s of every BASELINE.json config on one GPU (development report)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

R = rt.StereoRenderer(0)
res = {}
for name in ["C1", "C2", "C3", "C4", "C5"]:
    s = scenes.make_scene(name)
    info = R.upload(s)
    R.set_camera(s.rig)
    out = R.render(s.width, s.height, s.max_depth, count=True)
    torch.cuda.synchronize()
    c = R.counters_dict(out["counters"])
    rays = c["primary"] + c["reflection"] + c["refraction"] + c["shadow"]
    fb = R.alloc_fb(s.width, s.height)
    for _ in range(3):
        R.render(s.width, s.height, s.max_depth, fb=fb)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(20):
        ev[0].record()
        R.render(s.width, s.height, s.max_depth, fb=fb)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    ms = float(np.median(ts))
    res[name] = dict(ms=ms, fps=1e3 / ms, mrays_s=rays / ms / 1e3, rays=rays, counts=c, build_us=info["build_us"],
                     bvh_nodes=info["bvh_nodes"], bvh_depth=info["bvh_depth"], device_mb=info["device_bytes"] / 1e6)
    print(name, f"{ms:.3f} ms  {1e3/ms:.1f} fps  {rays/ms/1e3:.1f} Mrays/s  rays {rays}  build {info['build_us']/1e3:.1f} ms",
          flush=True)
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else "all_configs.json", "w"), indent=1)
