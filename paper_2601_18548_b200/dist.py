"""Multi-GPU gather of sharded active sets.

The obstacle points are sharded over ranks by 128-id block (block % world == rank,
gcdf_options.rank/world); every rank runs the fused detect over its own points, then:

  1. all_reduce(MIN) of the per-waypoint int64 keys  -> global min / argmin
  2. all_gather of the per-rank wp_offsets [n_wp + 1] -> every rank's block structure
  3. all_gather of the records, padded to the largest rank count (NCCL has no
     allgatherv; counts are balanced because blocks are dealt round-robin)
  4. gcdf_merge_active_sets (a CUDA kernel): canonical (wp, pt) order by merge-path
     binary search across the rank segments.

Steps 1-3 are torch.distributed collectives (NCCL over NVLink on B200 boxes, gloo in the
CPU tests); step 4 is the library's kernel.  No step computes on the host.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

REC_BYTES = 48


def gather_parts(local: dict, n_wp: int, group=None) -> dict:
    """Collectives only.  local: detect outputs of this rank (records uint8 [cap, 48],
    wp_offsets int64 [n_wp+1], wp_key int64 [n_wp]).  Returns the gathered pieces."""
    world = dist.get_world_size(group)
    key = local["wp_key"][:n_wp].clone()
    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    offs = torch.empty(world * (n_wp + 1), dtype=torch.int64, device=key.device)
    dist.all_gather_into_tensor(offs, local["wp_offsets"][: n_wp + 1].contiguous(), group=group)
    counts = offs.view(world, n_wp + 1)[:, n_wp]
    stride = int(counts.max().item())
    recs = local["records"]
    if recs.shape[0] < stride:
        recs = torch.cat([recs, recs.new_zeros((stride - recs.shape[0], REC_BYTES))])
    mine = recs[:stride].contiguous() if stride > 0 else recs.new_zeros((1, REC_BYTES))
    s = max(stride, 1)
    buf = torch.empty((world * s, REC_BYTES), dtype=torch.uint8, device=key.device)
    dist.all_gather_into_tensor(buf, mine if mine.shape[0] == s else mine[:s], group=group)
    return {"world": world, "n_wp": n_wp, "records": buf, "stride": s, "offsets": offs, "wp_key": key,
            "count": int(counts.sum().item())}


def gather_active_sets(ctx, local: dict, n_wp: int, capacity: int | None = None, group=None) -> dict:
    """Collectives + the merge kernel: the full, canonically ordered active set on every rank."""
    p = gather_parts(local, n_wp, group)
    cap = capacity if capacity is not None else max(p["count"], 1)
    out = ctx.merge_active_sets(p["world"], n_wp, p["records"], p["stride"], p["offsets"], p["wp_key"], cap)
    out["n"] = p["count"]
    return out
