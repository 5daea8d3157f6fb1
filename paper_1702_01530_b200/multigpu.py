"""Multi-GPU frames through the C ABI (SURVEY.md §8(a) row a7, §8(b) rt_dist_init, §8(e);
PAPER.md:48 "dividing the picture to N identical parts", PAPER.md:56 level-1 left/right channels).

The library does the sharding and the frame assembly (include/rt_b200.h, "multi-GPU frames"):
after rt_dist_init every rank's frame render traces that rank's tiles and rank 0's framebuffers
receive the whole frame -- by default through peer stores fused into the other ranks' pack
epilogues (CUDA IPC over NVLink, device-side completion flags), or by an NCCL gather + unpack.
Python only hands the 128-byte job id from rank 0 to the other ranks.
"""
from __future__ import annotations

from . import rt

TRANSPORTS = {"peer": rt.RT_DIST_PEER, "nccl": rt.RT_DIST_NCCL}


def join_world(R, rank, world, dist, transport="peer"):
    """Every rank joins the library's world: rank 0 creates the job id, torch.distributed
    broadcasts it (plumbing), rt_dist_init does the rest.  Returns rt_dist_info."""
    jid = [rt.rt_dist_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(jid, src=0)
    rt.rt_dist_init(R.ctx, rank, world, jid[0], TRANSPORTS[transport])
    return rt.rt_dist_info(R.ctx)


class Frame:
    """One stereo frame target.  Rank 0 (or a single GPU) renders into `fb` (2, H, W, 4); other
    ranks pass fb=None and their tiles land in rank 0's framebuffers."""

    def __init__(self, R, fb, width, height):
        self.R, self.fb, self.W, self.H = R, fb, width, height

    def render(self, depth, stream=None):
        self.R.render(self.W, self.H, depth, fb=self.fb if self.fb is not None else False, stream=stream)
