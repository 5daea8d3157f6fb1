"""Frames in flight on one GPU (development probe): per-frame throughput of K renders alternating
over F streams of ONE context (rt_render_stereo_async), for the full frame and for the shard one
GPU of an N-GPU run renders.  usage: python scripts/inflight_probe.py C4 [F ...]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

name = sys.argv[1]
depths = [int(x) for x in sys.argv[2:]] or [1, 2, 3, 4]
s = scenes.make_scene(name)
R = rt.StereoRenderer(0)
R.upload(s)
R.set_camera(s.rig)
streams = [torch.cuda.Stream() for _ in range(max(depths))]
fbs = [R.alloc_fb(s.width, s.height) for _ in range(max(depths))]
torch.cuda.synchronize()
K = 32
for world in (1, 2, 4, 8):
    for F in depths:
        worst = 0.0
        for rank in (0, world - 1):
            res = []
            for rep in range(2):
                torch.cuda.synchronize()
                st = torch.cuda.Event(enable_timing=True)
                st.record()
                for x in streams[:F]:
                    x.wait_event(st)
                for k in range(K):
                    R.render(s.width, s.height, s.max_depth, fb=fbs[k % F], shard=(rank, world), stream=streams[k % F])
                ends = []
                for x in streams[:F]:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(x)
                    ends.append(e)
                torch.cuda.synchronize()
                res.append(max(st.elapsed_time(e) for e in ends) / K)
            worst = max(worst, min(res))
        print(name, "world", world, "in flight", F, "ms/frame %.3f" % worst, flush=True)
