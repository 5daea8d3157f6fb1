import sys, torch, time, numpy as np
sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes
s = scenes.scene_c5(frame=0)
R = rt.StereoRenderer(0); R.upload(s)
F = 4
streams = [torch.cuda.Stream() for _ in range(F)]
fbs = [R.alloc_fb(s.width, s.height) for _ in range(F)]
rigs = [scenes.c5_rig(k) for k in range(60)]
rays = []
for rg in rigs[:60]:
    R.set_camera(rg); out = R.render(s.width, s.height, s.max_depth, fb=False, count=True); torch.cuda.synchronize()
    c = R.counters_dict(out["counters"]); rays.append(c["primary"]+c["reflection"]+c["refraction"]+c["shadow"])
print("mean rays/frame", np.mean(rays)/1e6, "frame0", rays[0]/1e6)
for mode in ("fixed", "orbit"):
    torch.cuda.synchronize(); st = torch.cuda.Event(enable_timing=True); st.record()
    for x in streams: x.wait_event(st)
    for k in range(60):
        R.set_camera(rigs[0] if mode == "fixed" else rigs[k])
        R.render(s.width, s.height, s.max_depth, fb=fbs[k % F], stream=streams[k % F])
    ends = []
    for x in streams:
        e = torch.cuda.Event(enable_timing=True); e.record(x); ends.append(e)
    torch.cuda.synchronize()
    ms = max(st.elapsed_time(e) for e in ends) / 60
    r = rays[0] if mode == "fixed" else np.mean(rays)
    print(mode, "%.3f ms/frame  %.0f Mrays/s" % (ms, r / ms / 1e3))
