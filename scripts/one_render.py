"""Render one C4 variant a few times (for ncu captures).  usage: one_render.py <depth> <n_lights>"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

depth, nl = int(sys.argv[1]), int(sys.argv[2])
base = scenes.scene_c4()
s = base.with_view(max_depth=depth)
s.lights = base.lights[:nl]
R = rt.StereoRenderer(0)
R.upload(s)
R.set_camera(s.rig)
fb = R.alloc_fb(s.width, s.height)
for _ in range(3):
    R.render(s.width, s.height, s.max_depth, fb=fb)
torch.cuda.synchronize()
