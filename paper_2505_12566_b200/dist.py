"""Request-sharded cascade across GPUs: forwarding deferred requests to the
ranks that hold the next stage's replicas.

The cascade's requests are independent, so the batch is sharded over
ranks (rank g owns a contiguous block of request ids).  After a stage, each
rank holds its deferred requests as a stable list (hs_route_compact).  The
next stage's batch is the GLOBAL stable deferred list -- rank-major
concatenation of the per-rank lists -- split into contiguous blocks over the
destination ranks R (the replicas of model m_{k+1}; "balanced" = all ranks):

    D_g = deferred count of rank g,  off_g = sum_{h<g} D_h,  D = sum_g D_g
    block i of R covers global positions [floor(i*D/|R|), floor((i+1)*D/|R|))

Because destinations are contiguous blocks of the global order, every rank
sends contiguous slices of its compacted buffers and every receiver gets its
block already in global order (chunks arrive in rank order).  The counts are
exchanged with an all-gather, the ids/payload with one all-to-all
(torch.distributed over NCCL on GPUs; gloo in the CPU tests).  The paper's
data movement between models is RPC/DMA; on an NVSwitch box it is
one NCCL all-to-all per stage.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def block_bounds(total: int, parts: int) -> list[int]:
    """lo_0..lo_parts with lo_i = floor(i * total / parts)."""
    return [(i * total) // parts for i in range(parts + 1)]


def exchange_plan(counts: list[int], dest_ranks: list[int], world: int) -> list[list[int]]:
    """send[g][h] = how many of rank g's deferred requests go to rank h."""
    total = sum(counts)
    lo = block_bounds(total, len(dest_ranks))
    send = [[0] * world for _ in range(world)]
    off = 0
    for g, d in enumerate(counts):
        a, b = off, off + d
        for i, h in enumerate(dest_ranks):
            s, e = max(a, lo[i]), min(b, lo[i + 1])
            if e > s:
                send[g][h] += e - s
        off = b
    return send


def forward_deferred(ids: torch.Tensor, count: torch.Tensor, *, dest_ranks: list[int] | None = None,
                     payload: torch.Tensor | None = None, group=None):
    """Move this rank's deferred requests (ids[:count], payload rows) to the
    next stage's ranks.  ``count`` is a 1-element int64 tensor on ids' device
    (d_counts[1] of hs_cascade_step).  Returns (recv_ids, recv_payload, n_recv).

    One device->host read of the gathered counts per stage: NCCL's all-to-all
    takes host split sizes."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dest = list(range(world)) if dest_ranks is None else list(dest_ranks)
    cnt = count.reshape(1).to(torch.int64)
    gathered = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(gathered, cnt, group=group)
    counts = [int(x.item()) for x in gathered]
    plan = exchange_plan(counts, dest, world)
    send = plan[rank]
    recv = [plan[g][rank] for g in range(world)]
    n_recv = sum(recv)
    out_ids = torch.empty(n_recv, dtype=ids.dtype, device=ids.device)
    dist.all_to_all_single(out_ids, ids[: counts[rank]].contiguous(), recv, send, group=group)
    out_payload = None
    if payload is not None:
        P = payload.shape[1]
        out_payload = torch.empty(n_recv, P, dtype=payload.dtype, device=payload.device)
        dist.all_to_all_single(out_payload, payload[: counts[rank]].contiguous(), recv, send,
                               group=group)
    return out_ids, out_payload, n_recv


def global_order_offsets(counts: list[int]) -> list[int]:
    """off_g = sum_{h<g} D_h: where rank g's deferred list starts in the global order."""
    off, acc = [], 0
    for d in counts:
        off.append(acc)
        acc += d
    return off
