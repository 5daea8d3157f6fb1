"""Dump a GPU render (fb, ids, radiance) of a config to npz for offline analysis.
usage: dump_gpu.py <config> <out.npz> [width height depth]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

s = scenes.make_scene(sys.argv[1])
if len(sys.argv) > 3:
    s = s.with_view(width=int(sys.argv[3]), height=int(sys.argv[4]), max_depth=int(sys.argv[5]))
R = rt.StereoRenderer(0)
R.upload(s)
R.set_camera(s.rig)
out = R.render(s.width, s.height, s.max_depth, want_id=True, want_radiance=True)
torch.cuda.synchronize()
np.savez_compressed(sys.argv[2], fb=out["fb"].cpu().numpy(), id=out["id"].cpu().numpy(),
                    radiance=out["radiance"].cpu().numpy())
print("saved", sys.argv[2])
