"""Multi-GPU upper-hood build: contiguous x-slabs, one exchange step.

SURVEY.md §8(e).  The x-sorted input shards naturally: rank r owns a
contiguous x-slab, builds that slab's hood on its own GPU (the ring kernel +
finalize, no collective), and the small slab hoods are exchanged once and
merged.  upper_hull(concat of slab hulls) == upper_hull(all points) because
every corner of the global hood is a corner of its slab's hood (a point
popped by the slab's monotone chain lies below a chord of two slab points,
oracle.cpp:7-20) -- the same argument the reference's round loop relies on
when it merges adjacent blocks (driver.cpp:20-43, kernel.cpp:117-137).

Exchange protocol (one collective in the common case):
  * every rank packs a fixed-size record  [count, pad | CAP corners]  in
    float64 (exact for float2 and double2 inputs), shifted by the slab's
    x offset into global coordinates;
  * all_gather of the records (NCCL over NVLink/NVSwitch on GPUs; gloo in the
    CPU tests);
  * if some slab hood has more than CAP corners (arc-like slabs), a second,
    count-sized all_gather carries the full hoods;
  * every rank merges the G slab hoods with hood_merge_segments (GPU) --
    ranks end with identical global hoods, no broadcast needed.

The device operations are injected as callables so the host-side protocol is
tested on CPU with gloo (tests/test_distributed.py); the defaults are the CUDA
path and fail loudly without it.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

DEFAULT_CAP = 4096


def slab_range(n_global: int, world: int, rank: int, block_len: int = 0):
    """[lo, hi) of rank's contiguous x-slab of ONE global x-sorted set of
    n_global points (contiguous slabs of n/G, G a power of
    two, so slabs are reference round-blocks); batched sets (block_len > 0)
    split on instance boundaries.  The slab keeps its global coordinates, so
    the exchange needs no x offset (exact for double2 as well as float2)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    unit = block_len if block_len else 1
    if n_global % unit:
        raise ValueError("n_global must be a multiple of block_len")
    units = n_global // unit
    if units % world:
        raise ValueError(f"{units} {'instances' if block_len else 'points'} do not split over {world} ranks")
    per = units // world
    return rank * per * unit, (rank + 1) * per * unit


@dataclass
class ShardResult:
    hull: "object"          # (k, 2) float64 tensor: the global hood, left to right
    slab_counts: list       # corners of every rank's slab hood
    exchanges: int          # collectives used (1, or 2 on record overflow)


def pack_record(corners, count: int, cap: int, x_offset: float = 0.0):
    """(cap + 1, 2) float64 record: row 0 = (count, 0), rows 1.. = corners."""
    import torch

    rec = torch.zeros(cap + 1, 2, dtype=torch.float64, device=corners.device)
    k = min(int(count), cap)
    if k:
        h = corners[:k].to(torch.float64, copy=True)
        if x_offset:
            h[:, 0] += x_offset
        rec[1:k + 1] = h
    rec[0, 0] = float(count)
    return rec


def _gather(t, group=None):
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return torch.stack(out)


def sharded_build_device(points, corners, counts, rec, gathered, out, out_count, x_offset: float = 0.0,
                         group=None, block_len: int = 0):
    """The graph-capturable form used by bench.py: build this rank's slab hood
    into (corners, counts), pack it (hood_pack_record), all-gather the records
    over NCCL and merge them (hood_merge_records) -- no host synchronisation.
    rec (cap+1, 2), gathered (G, cap+1, 2), out (G*cap, 2) float64 buffers."""
    import torch.distributed as dist

    from . import hood as H

    H.build_hood_async(points, block_len, corners=corners, counts=counts)
    H.pack_record(corners, counts, rec.shape[0] - 1, x_offset=x_offset, rec=rec)
    dist.all_gather_into_tensor(gathered.view(-1), rec.view(-1), group=group)
    H.merge_records(gathered, out=out, out_count=out_count)
    return out, out_count


def merge_gpu(seg_pts, seg_counts):
    """hood_merge_segments over (G, stride, 2) float64 slab hoods."""
    import torch

    from . import hood as H

    out, cnt = H.merge_segments(seg_pts.contiguous(), seg_counts.to(device=seg_pts.device, dtype=torch.int32))
    return out[: int(cnt.item())]


def build_local_gpu(points, block_len: int = 0):
    """Slab hood on this rank's GPU: (corners tensor, count)."""
    from . import hood as H

    rep = H.build_hood(points)
    return rep.hull, len(rep.hull)


def sharded_build(points, group=None, cap: int = DEFAULT_CAP, x_offset: float = 0.0,
                  build_local: Optional[Callable] = None, merge: Optional[Callable] = None) -> ShardResult:
    """Global upper hood of the x-slabs held by the ranks of `group`.

    points   this rank's slab, (n_r, 2), x strictly increasing, every x left of
             the next rank's slab (after adding x_offset).
    x_offset added to this rank's x in float64 to form global x: exact for
             float2 slabs (a float widened to double plus a small integer);
             double2 slabs should be cut from one global set (slab_range) and
             use offset 0, as bench.py does.
    """
    import torch

    build_local = build_local or build_local_gpu
    merge = merge or merge_gpu
    corners, count = build_local(points)
    rec = pack_record(corners, count, cap, x_offset)
    recs = _gather(rec, group)                                  # (G, cap + 1, 2)
    counts = recs[:, 0, 0].to(torch.int64).tolist()
    exchanges = 1
    if max(counts) > cap:
        # a slab hood overflowed the record: one more exchange, sized exactly
        big = max(counts)
        full = torch.zeros(big, 2, dtype=torch.float64, device=corners.device)
        if count:
            h = corners[:count].to(torch.float64, copy=True)
            if x_offset:
                h[:, 0] += x_offset
            full[:count] = h
        segs = _gather(full, group)
        exchanges = 2
    else:
        segs = recs[:, 1:, :]
    seg_counts = torch.tensor(counts, dtype=torch.int32, device=segs.device)
    hull = merge(segs, seg_counts)
    return ShardResult(hull=hull, slab_counts=counts, exchanges=exchanges)
