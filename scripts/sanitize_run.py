"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
upload + BVH build (spheres, planes, triangles; a 90k-triangle mesh for the CTA-level SAH tasks),
stereo renders with every output, the fused composition, shards + device unpack (round-robin and
block layouts are separate processes: RT_SHARD_BLOCK), refit, compose, download, B0 probes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402

R = rt.StereoRenderer(0)
for s in (scenes.scene_c1(), scenes.scene_c2().with_view(width=40, height=30, max_depth=3),
          scenes.scene_c3().with_view(width=48, height=27), scenes.scene_c4(nu=300, nv=150).with_view(width=40, height=24)):
    R.upload(s)
    R.set_camera(s.rig)
    out = R.render(s.width, s.height, s.max_depth, want_id=True, want_radiance=True, count=True)
    R.render(s.width, s.height, s.max_depth, fmt=rt.RT_FORMAT_RGBA16F)
    for world in (2, 3):
        per = rt.rt_shard_bytes(s.width, s.height, world)
        g = torch.zeros(world * per, dtype=torch.uint8, device="cuda")
        for r in range(world):
            R.render(s.width, s.height, s.max_depth, fb=False, shard=(r, world), shard_buf=g[r * per:(r + 1) * per])
        fb = torch.zeros((2, s.height, s.width, 4), dtype=torch.uint8, device="cuda")
        rt.rt_unpack_shards(R.ctx, g.data_ptr(), s.width, s.height, world, 0,
                            rt.rt_fb(fb[0].data_ptr(), 0, s.width * 4), rt.rt_fb(fb[1].data_ptr(), 0, s.width * 4))
    rt.rt_kdtree_build(R.ctx, 2, 0)                      # NEXT-4 kd-tree ablation kernel
    R.render(s.width, s.height, s.max_depth, want_id=True, kdtree=True)
    if s.n_tris:
        rt.rt_scene_update_vertices(R.ctx, s.vertices * 1.01)
        R.render(s.width, s.height, s.max_depth)
    for mode in (rt.RT_COMPOSE_ANAGLYPH, rt.RT_COMPOSE_SBS):
        c = torch.zeros((s.height, s.width if mode == 0 else 2 * (s.width // 2), 4), dtype=torch.uint8, device="cuda")
        R.render(s.width, s.height, s.max_depth, compose=(mode, c))
    f = out["fb"]
    o = torch.zeros((s.height, s.width, 4), dtype=torch.uint8, device="cuda")
    rt.rt_compose(R.ctx, rt.rt_fb(f[0].data_ptr(), 0, s.width * 4), rt.rt_fb(f[1].data_ptr(), 0, s.width * 4),
                  s.width, s.height, 0, rt.rt_fb(o.data_ptr(), 0, s.width * 4))
    h = rt.rt_host_alloc(f.numel())
    rt.rt_wait(rt.rt_download(R.ctx, f.data_ptr(), h, f.numel()))
    rt.rt_host_free(h)
rt.rt_bench_ceilings(R.ctx)
torch.cuda.synchronize()
R.close()
print("sanitize workload done")
