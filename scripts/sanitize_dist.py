"""Two ranks on one GPU through rt_dist_init (peer transport) for compute-sanitizer
(--target-processes all): the slot post / completion wait / signal kernels and the peer-store
epilogue into the other process's framebuffers."""
import os
import socket
import sys

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1702_01530_b200 import multigpu, rt, scenes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = scenes.scene_c2().with_view(width=40, height=30, max_depth=2)
    R = rt.StereoRenderer(0)
    R.upload(s)
    R.set_camera(s.rig)
    multigpu.join_world(R, rank, world, dist)
    for _ in range(3):
        fb = R.alloc_fb(s.width, s.height) if rank == 0 else None
        multigpu.Frame(R, fb, s.width, s.height).render(s.max_depth)
    torch.cuda.synchronize()
    rt.rt_dist_finalize(R.ctx)
    dist.barrier()
    R.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    mp.spawn(worker, args=(2, port), nprocs=2)
    print("sanitize dist workload done")
