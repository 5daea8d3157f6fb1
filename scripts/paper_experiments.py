"""NEXT-2: the structure of the paper's experiments (§4, Figs. 3-8) on one B200.

* Figs. 3-6 / §5 "dependence has almost linear character": synthesis time vs scene complexity
  for SPEC's paper scenes (1, 2, 3, 5, 6 polyhedra, 1 light), split into transfer-in (scene
  upload + BVH build), compute (stereo render) and transfer-out (pinned download).
* Fig. 7: stage fractions of the 6-object scene (paper: ~60 % compute, up to 40 % transfer).
* Fig. 8 / P:109 "network size": compute time vs the number of trace CTAs (RT_GRID_LIMIT),
  the B200 analogue of the paper's (B:T) CUDA network configurations ((4:1) vs (1:1) = 2.5x).
Writes a CSV (SPEC.md:565-style columns) and a JSON summary.
usage: python scripts/paper_experiments.py <out_prefix>
"""
import csv
import json
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, ".")

W = H = 512
DEPTH = 3


def stage_run(n_objects, reps=5):
    import torch

    from paper_1702_01530_b200 import rt, scenes
    s = scenes.paper_scene(n_objects).with_view(width=W, height=H, max_depth=DEPTH)
    R = rt.StereoRenderer(0)
    nbytes = 2 * H * W * 4
    host = rt.rt_host_alloc(nbytes)
    fb = R.alloc_fb(W, H)
    rows = []
    for rep in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        R.upload(s)                                  # transfer-in: host arrays -> device + BVH build
        R.set_camera(s.rig)
        t1 = time.perf_counter()
        R.render(W, H, DEPTH, fb=fb)
        rt.rt_synchronize(R.ctx)
        t2 = time.perf_counter()
        rt.rt_wait(rt.rt_download(R.ctx, fb.data_ptr(), host, nbytes))
        t3 = time.perf_counter()
        rows.append(dict(scene_id=f"paper{n_objects}", objects=n_objects, triangles=s.n_tris, width=W, height=H,
                         rep=rep, transfer_in_ns=int((t1 - t0) * 1e9), compute_ns=int((t2 - t1) * 1e9),
                         transfer_out_ns=int((t3 - t2) * 1e9), total_ns=int((t3 - t0) * 1e9)))
    rt.rt_host_free(host)
    R.close()
    return rows


def grid_run(limit):
    env = dict(os.environ, RT_GRID_LIMIT=str(limit))
    code = ("import sys,torch,numpy as np;sys.path.insert(0,'.');from paper_1702_01530_b200 import rt,scenes;"
            f"s=scenes.paper_scene(6).with_view(width={W},height={H},max_depth={DEPTH});R=rt.StereoRenderer(0);"
            "R.upload(s);R.set_camera(s.rig);fb=R.alloc_fb(s.width,s.height);"
            "[R.render(s.width,s.height,s.max_depth,fb=fb) for _ in range(3)];torch.cuda.synchronize();"
            "e=[torch.cuda.Event(enable_timing=True) for _ in range(2)];ts=[]\n"
            "for _ in range(7):\n e[0].record();R.render(s.width,s.height,s.max_depth,fb=fb);e[1].record();"
            "torch.cuda.synchronize();ts.append(e[0].elapsed_time(e[1]))\n"
            "print(float(np.median(ts)))")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    return float(out.stdout.strip().splitlines()[-1])


def main():
    prefix = sys.argv[1] if len(sys.argv) > 1 else "paper_experiments"
    rows = []
    for n in (1, 2, 3, 5, 6):
        rows += stage_run(n)
    with open(prefix + ".csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    summary = {"resolution": f"{W}x{H} per eye", "depth": DEPTH, "complexity": {}, "grid": {}}
    for n in (1, 2, 3, 5, 6):
        rs = [r for r in rows if r["objects"] == n and r["rep"] > 0]
        med = {k: float(np.median([r[k] for r in rs])) / 1e6 for k in ("transfer_in_ns", "compute_ns", "transfer_out_ns",
                                                                        "total_ns")}
        tot = med["transfer_in_ns"] + med["compute_ns"] + med["transfer_out_ns"]
        med.update(triangles=rs[0]["triangles"], compute_fraction=med["compute_ns"] / tot,
                   transfer_fraction=(med["transfer_in_ns"] + med["transfer_out_ns"]) / tot)
        summary["complexity"][f"paper{n}"] = med
        print(f"paper{n}: {rs[0]['triangles']:4d} tris  in {med['transfer_in_ns']:.3f} ms  compute {med['compute_ns']:.3f} ms"
              f"  out {med['transfer_out_ns']:.3f} ms  compute fraction {med['compute_fraction']:.2f}", flush=True)
    for limit in (1, 2, 4, 8, 16, 37, 74, 148, 296, 592, 1184, 2368):
        ms = grid_run(limit)
        summary["grid"][limit] = ms
        print(f"trace CTAs {limit:4d}: {ms:.3f} ms", flush=True)
    g = summary["grid"]
    summary["speedup_4_vs_1_cta"] = g[1] / g[4]
    summary["speedup_4_vs_2_cta"] = g[2] / g[4]
    summary["speedup_full_vs_1_cta"] = g[1] / min(g.values())
    summary["paper"] = {"4:1 vs 1:1": 2.5, "4:1 vs 2:1": "20-25 % less time", "compute_fraction": 0.6,
                        "transfer_fraction": "up to 0.4", "source": "PAPER.md:15, :106-109; unnamed NVIDIA GPU (P:66)"}
    json.dump(summary, open(prefix + ".json", "w"), indent=1)


if __name__ == "__main__":
    main()
