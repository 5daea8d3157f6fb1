import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes
R = rt.StereoRenderer(0)
flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for name in sys.argv[1:]:
    s = scenes.make_scene(name)
    R.upload(s); R.set_camera(s.rig)
    fb = R.alloc_fb(s.width, s.height)
    for depth in (s.max_depth, 0):
        for world in (1, 8, 64, 512, 4096):
            ts = []
            for rank in (0, world // 3, world // 2):
                for i in range(6):
                    flush.zero_(); ev[0].record()
                    R.render(s.width, s.height, depth, fb=fb, shard=(rank, world))
                    ev[1].record(); torch.cuda.synchronize()
                    if i >= 2: ts.append(ev[0].elapsed_time(ev[1]))
            print(name, "depth", depth, "world", world, "median ms %.3f max %.3f" % (np.median(ts), max(ts)), flush=True)
