"""Multi-GPU plumbing for the STL layer.

* Forward: token rows (M) shard with no collective — rows of Y depend only on the same rows of
  X and on the replicated (W_enc, e_x, d) (snf_operator.py:146-152). ``shard_rows`` gives each
  rank a contiguous slab whose size is a multiple of the tile size t.
* Data-parallel training: each rank runs the layer step on its own batch; the only exchange is
  an all-reduce of the gradients (g_w, g_ex, g_d). ``GradBucket`` packs them into one flat fp32
  buffer so the exchange is a single NCCL call (bucketed for launch latency, not link count —
  every GPU sees every peer at full NVLink bandwidth through NVSwitch).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(M: int, t: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """[start, stop) token rows owned by `rank`; boundaries are multiples of t*align tiles."""
    if M % t:
        raise ValueError(f"M={M} is not a multiple of the tile size t={t}")
    unit = t * max(align, 1)
    units = -(-M // unit)
    per, extra = divmod(units, world)
    lo = rank * per + min(rank, extra)
    hi = lo + per + (1 if rank < extra else 0)
    return min(lo * unit, M), min(hi * unit, M)


class GradBucket:
    """One flat fp32 buffer with views for an STL layer's three gradients."""

    def __init__(self, r: int, t: int, out_tiles: int, in_tiles: int, device):
        nw = r * out_tiles * in_tiles
        ne = r * t * t
        self.flat = torch.zeros(nw + 2 * ne, dtype=torch.float32, device=device)
        self.g_w = self.flat[:nw].view(r, out_tiles, in_tiles)   # native planes layout
        self.g_ex = self.flat[nw:nw + ne].view(r, t * t)
        self.g_d = self.flat[nw + ne:].view(r, t * t)

    def allreduce(self, group=None, average: bool = False) -> None:
        dist.all_reduce(self.flat, group=group)
        if average:
            self.flat /= dist.get_world_size(group)


def allreduce_grads(tensors, group=None) -> None:
    """Bucketed all-reduce of arbitrary gradient tensors (pack, one collective, unpack)."""
    tensors = [t for t in tensors if t is not None]
    if not tensors:
        return
    dtype = tensors[0].dtype if all(t.dtype == tensors[0].dtype for t in tensors) else torch.float32
    flat = torch.cat([t.reshape(-1).to(dtype) for t in tensors])
    dist.all_reduce(flat, group=group)
    off = 0
    for t in tensors:
        n = t.numel()
        t.copy_(flat[off:off + n].view_as(t))
        off += n
