"""Multi-GPU frame assembly ("dividing the picture
to N identical parts", PAPER.md:56 level-1 left/right channels).

Every rank holds the whole scene (deterministic LBVH, identical on every rank) and renders only
its tiles (rt_shard_tiles: world 2 = eye split, otherwise 16x16 tiles dealt round-robin, both
eyes of a tile to the same rank).  Two ways to assemble the frame on rank 0:

  "peer"  fused render -> gather: rank 0 exports its framebuffers with CUDA IPC, every other
          rank maps them (rt_ipc_open) and its trace kernel's pack epilogue stores its tiles
          straight into rank 0's framebuffers over NVLink (RT_RENDER_PEER_STORE: system fence
          at kernel exit).  One barrier closes the frame.  No gather call, no unpack kernel.
  "nccl"  each rank packs its tiles into a contiguous shard, torch.distributed.gather (NCCL
          send/recv over NVLink) brings them to rank 0, k_unpack_shards scatters them.

PyTorch supplies only the process group (plumbing); the data path is the library's kernels.
"""
from __future__ import annotations

from . import rt


def gather_to_root(dist, shard_buf, gathered, world, rank, per):
    """a7 (nccl path): every rank's packed tile shard -> rank 0's `gathered` (rank-major)."""
    glist = [gathered[r * per:(r + 1) * per] for r in range(world)] if rank == 0 else None
    dist.gather(shard_buf, glist, dst=0)


class NcclFrame:
    """Shard render + gather + root unpack."""

    mode = "nccl"
    pipelined = False        # gather + unpack are collective calls per frame: frames run one at a time

    def __init__(self, R, fb, rank, world, dist, width, height):
        import torch
        self.R, self.fb, self.rank, self.world, self.dist = R, fb, rank, world, dist
        self.W, self.H = width, height
        self.per = rt.rt_shard_bytes(width, height, world)
        self.shard = torch.empty(self.per, dtype=torch.uint8, device=R.device)
        self.gathered = torch.empty(world * self.per, dtype=torch.uint8, device=R.device) if rank == 0 else None
        self.launches_per_frame = 1 + (1 if rank == 0 else 0)

    def render(self, depth, stream=None):
        assert stream is None, "the NCCL gather path renders one frame at a time"
        self.R.render(self.W, self.H, depth, fb=False, shard=(self.rank, self.world), shard_buf=self.shard)

    def assemble(self):
        gather_to_root(self.dist, self.shard, self.gathered, self.world, self.rank, self.per)
        if self.rank == 0:
            pitch = self.W * 4
            rt.rt_unpack_shards(self.R.ctx, self.gathered.data_ptr(), self.W, self.H, self.world, rt.RT_FORMAT_RGBA8,
                                rt.rt_fb(self.fb[0].data_ptr(), 0, pitch), rt.rt_fb(self.fb[1].data_ptr(), 0, pitch))

    def close(self):
        pass


class PeerFrame:
    """Fused render -> gather through rank 0's IPC-mapped framebuffers."""

    mode = "peer"
    pipelined = True         # frames in flight: each slot has its own mapped framebuffers

    def __init__(self, R, fb, rank, world, dist, width, height):
        self.R, self.rank, self.world, self.dist = R, rank, world, dist
        self.W, self.H = width, height
        handle = [rt.rt_ipc_get_handle(fb.data_ptr()) if rank == 0 else None]
        dist.broadcast_object_list(handle, src=0)
        self.mapped = None
        if rank == 0:
            base = fb.data_ptr()
        else:
            h, offset = handle[0]
            self.mapped = rt.rt_ipc_open(R.ctx, h)
            base = self.mapped + offset
        self.ptrs = (base, base + height * width * 4, width * 4)      # (2, H, W, 4) u8 layout
        self.launches_per_frame = 1

    def render(self, depth, stream=None):
        self.R.render(self.W, self.H, depth, fb_ptrs=self.ptrs, shard=(self.rank, self.world), peer=self.rank != 0,
                      stream=stream)

    def assemble(self):
        self.dist.barrier()           # every rank's stores have landed in rank 0's framebuffers

    def close(self):
        if self.mapped:
            rt.rt_ipc_close(self.R.ctx, self.mapped)
            self.mapped = None


def make_frame(mode, R, fb, rank, world, dist, width, height):
    if mode == "peer":
        try:
            f = PeerFrame(R, fb, rank, world, dist, width, height)
            ok = 1
        except rt.RtError:
            f, ok = None, 0
        import torch
        flag = torch.tensor([ok], dtype=torch.int32, device=R.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            return f
        if f is not None:
            f.close()
    return NcclFrame(R, fb, rank, world, dist, width, height)
