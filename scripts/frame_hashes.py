"""SHA-256 of the rendered outputs (RGBA8 framebuffers, primary IDs, FP32 radiance) of every
BASELINE config, for bit-identity checks between two builds of the library (RT_LIB_PATH).

    RT_LIB_PATH=... python scripts/frame_hashes.py out.json
"""
import hashlib
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

R = rt.StereoRenderer(0)
res = {}
for name in ["C1", "C2", "C3", "C4", "C5"]:
    s = scenes.make_scene(name)
    R.upload(s)
    R.set_camera(s.rig)
    out = R.render(s.width, s.height, s.max_depth, want_id=True, want_radiance=True)
    torch.cuda.synchronize()
    res[name] = {k: hashlib.sha256(out[k].cpu().numpy().tobytes()).hexdigest()[:16] for k in ("fb", "id", "radiance")}
    print(name, res[name], flush=True)
json.dump(res, open(sys.argv[1], "w"), indent=1)
