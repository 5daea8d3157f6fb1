"""Predicted strong scaling from per-shard kernel times on ONE B200 (this run has one GPU).

For world = 1, 2, 4, 8 every rank's shard (rt_render_stereo_ex with shard (rank, world), the
launch the N-GPU bench makes on each GPU) is rendered alone on the whole device, L2 flushed
before each frame: one frame at a time (median of 7) and, as the bench's throughput loop runs
it, RT_INFLIGHT (4) frames in flight on separate streams.  The slowest shard bounds an N-GPU
step (plus the frame barrier, not modelled here); predicted speedup = T(1) / max_rank T(rank, world).
usage: python scripts/shard_scaling.py [C4 ...] > out.json
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_01530_b200 import rt, scenes  # noqa: E402


NOFLUSH = os.environ.get("RT_NOFLUSH") == "1"   # warm-L2 comparison only (the bench always flushes)
INFLIGHT = int(os.environ.get("RT_INFLIGHT", "4"))
K_FRAMES = int(os.environ.get("RT_K", "24"))        # frames per pipelined measurement (the drain is amortised over K)


def main():
    names = sys.argv[1:] or ["C4"]
    R = rt.StereoRenderer(0)
    # the bench's flush (bench.l2_flush_bytes: 1.25x L2, at least 160 MiB) unless RT_FLUSH_MIB overrides it
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import l2_flush_bytes
    fb_bytes = int(os.environ["RT_FLUSH_MIB"]) << 20 if "RT_FLUSH_MIB" in os.environ else l2_flush_bytes(torch.device("cuda", 0))
    flush = torch.empty(fb_bytes // 4, dtype=torch.float32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    res = {}
    for name in names:
        s = scenes.make_scene(name)
        R.upload(s)
        R.set_camera(s.rig)
        fb = R.alloc_fb(s.width, s.height)
        rows = {}
        streams = [torch.cuda.Stream() for _ in range(INFLIGHT)]
        fbs = [fb] + [R.alloc_fb(s.width, s.height) for _ in range(INFLIGHT - 1)]
        for world in (1, 2, 4, 8):
            per_rank, per_rank_pipe = [], []
            for rank in range(world):
                ts = []
                for i in range(10):
                    if not NOFLUSH:
                        flush.zero_()
                    ev[0].record()
                    R.render(s.width, s.height, s.max_depth, fb=fb, shard=(rank, world))
                    ev[1].record()
                    torch.cuda.synchronize()
                    if i >= 3:
                        ts.append(ev[0].elapsed_time(ev[1]))
                per_rank.append(float(np.median(ts)))
                # the bench's throughput regime: INFLIGHT frames in flight, flush before each
                K = K_FRAMES
                for rep in range(2):
                    torch.cuda.synchronize()
                    st = torch.cuda.Event(enable_timing=True)
                    st.record()
                    for x in streams:
                        x.wait_event(st)
                    for k in range(K):
                        x = streams[k % INFLIGHT]
                        with torch.cuda.stream(x):
                            if not NOFLUSH:
                                flush.zero_()
                        R.render(s.width, s.height, s.max_depth, fb=fbs[k % INFLIGHT], shard=(rank, world), stream=x)
                    ends = []
                    for x in streams:
                        e = torch.cuda.Event(enable_timing=True)
                        e.record(x)
                        ends.append(e)
                    torch.cuda.synchronize()
                    if rep:
                        per_rank_pipe.append(max(st.elapsed_time(e) for e in ends) / K)
            rows[world] = {"ms_per_rank": per_rank, "max_ms": max(per_rank), "mean_ms": float(np.mean(per_rank)),
                           "pipelined_ms_per_rank": per_rank_pipe, "pipelined_max_ms": max(per_rank_pipe)}
        t1 = rows[1]["max_ms"]
        p1 = rows[1]["pipelined_max_ms"]
        for world, r in rows.items():
            r["predicted_speedup"] = t1 / r["max_ms"]
            r["predicted_efficiency"] = t1 / (world * r["max_ms"])
            r["imbalance_max_over_mean"] = r["max_ms"] / r["mean_ms"]
            r["pipelined_predicted_speedup"] = p1 / r["pipelined_max_ms"]
            r["pipelined_predicted_efficiency"] = p1 / (world * r["pipelined_max_ms"])
            print(name, world, f"one frame: max {r['max_ms']:.3f} ms  speedup {r['predicted_speedup']:.2f}  "
                  f"imbalance {r['imbalance_max_over_mean']:.3f} | {INFLIGHT} in flight: {r['pipelined_max_ms']:.3f} ms "
                  f"speedup {r['pipelined_predicted_speedup']:.2f}", file=sys.stderr)
        res[name] = rows
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
