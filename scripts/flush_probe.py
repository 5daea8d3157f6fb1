import sys, torch
sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes
s = scenes.make_scene("C4")
R = rt.StereoRenderer(0); R.upload(s); R.set_camera(s.rig)
F = 4
streams = [torch.cuda.Stream() for _ in range(F)]
fbs = [R.alloc_fb(s.width, s.height) for _ in range(F)]
nb = 160 << 20
flush = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
zsrc = torch.zeros_like(flush)
def run(world, rank, mode, K=24):
    res = []
    for rep in range(2):
        torch.cuda.synchronize()
        st = torch.cuda.Event(enable_timing=True); st.record()
        for x in streams: x.wait_event(st)
        for k in range(K):
            x = streams[k % F]
            with torch.cuda.stream(x):
                if mode == "kernel": flush.zero_()
                elif mode == "copy": flush.copy_(zsrc, non_blocking=True)
            R.render(s.width, s.height, s.max_depth, fb=fbs[k % F], shard=(rank, world), stream=x)
        ends = []
        for x in streams:
            e = torch.cuda.Event(enable_timing=True); e.record(x); ends.append(e)
        torch.cuda.synchronize()
        res.append(max(st.elapsed_time(e) for e in ends) / K)
    return min(res)
for world in (1, 8):
    for mode in ("none", "kernel", "copy"):
        print(world, mode, "%.3f ms/frame" % max(run(world, r, mode) for r in (0, world - 1)), flush=True)
