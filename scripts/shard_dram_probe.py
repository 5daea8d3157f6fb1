"""Per-shard DRAM traffic of the world-8 tile layout (run under ncu, whose default cache control
flushes L2 before every kernel -- the bench's cold-L2 condition):
    RT_SHARD_BLOCK=B ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:k_trace_stereo --csv python scripts/shard_dram_probe.py [C4] [world]
Each rank's shard of one frame is rendered once (the launch an N-GPU run makes on each GPU)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
s = scenes.make_scene(name)
R = rt.StereoRenderer(0)
R.upload(s)
R.set_camera(s.rig)
fb = R.alloc_fb(s.width, s.height)
R.render(s.width, s.height, s.max_depth, fb=fb)          # whole frame first (reference launch)
for r in range(world):
    R.render(s.width, s.height, s.max_depth, fb=fb, shard=(r, world))
torch.cuda.synchronize()
