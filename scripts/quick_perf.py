"""Quick timing of one config (development aid; bench.py is the contract)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
t0 = time.time()
s = scenes.make_scene(name)
print(f"scene {name} gen {time.time()-t0:.1f}s tris {s.n_tris} spheres {s.n_spheres}", flush=True)
R = rt.StereoRenderer(0)
t0 = time.time()
info = R.upload(s)
print("upload", f"{time.time()-t0:.2f}s", info, flush=True)
R.set_camera(s.rig)
out = R.render(s.width, s.height, s.max_depth, count=True)
torch.cuda.synchronize()
c = R.counters_dict(out["counters"])
print(c)
rays = c["primary"] + c["reflection"] + c["refraction"] + c["shadow"]
fb = R.alloc_fb(s.width, s.height)
for _ in range(3):
    R.render(s.width, s.height, s.max_depth, fb=fb)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(10):
    ev[0].record()
    R.render(s.width, s.height, s.max_depth, fb=fb)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ts.sort()
ms = ts[len(ts) // 2]
print(f"{name}: median {ms:.3f} ms/stereo frame, {rays/ms/1e3:.1f} Mrays/s, rays/frame {rays}, fps {1e3/ms:.1f}")
# frames in flight like bench.py: F = 4 streams, L2 flush (160 MiB write) before every frame
F, K = 4, 40
streams = [torch.cuda.Stream() for _ in range(F)]
fbs = [R.alloc_fb(s.width, s.height) for _ in range(F)]
flush = [torch.empty(160 << 20, dtype=torch.uint8, device="cuda") for _ in range(F)]
best = 1e9
for rep in range(3):
    torch.cuda.synchronize()
    st = torch.cuda.Event(enable_timing=True)
    st.record()
    for x in streams:
        x.wait_event(st)
    for k in range(K):
        with torch.cuda.stream(streams[k % F]):
            flush[k % F].fill_(k & 255)
        R.render(s.width, s.height, s.max_depth, fb=fbs[k % F], stream=streams[k % F])
    ends = []
    for x in streams:
        e = torch.cuda.Event(enable_timing=True)
        e.record(x)
        ends.append(e)
    torch.cuda.synchronize()
    best = min(best, max(st.elapsed_time(e) for e in ends) / K)
print(f"{name}: inflight {best:.3f} ms/stereo frame, {rays/best/1e3:.1f} Mrays/s")
