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


class _DevArray:
    """A torch view of a raw device allocation (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class PeerForwarder:
    """Forwarding of deferred requests over peer memory (hs_forward_*): the
    same result as :func:`forward_deferred` -- this rank's block of the global
    stable deferred list -- moved by the kernels through CUDA IPC mappings of
    the peers' buffers (NVLink / NVSwitch), with no host round trip and no NCCL
    on the data path.  The IPC handles are exchanged once, at construction,
    with ``all_gather_object`` over the process group.

    Buffers per rank (one exportable allocation each, hs_ipc_alloc): the count
    and done flag arrays (u64[world]) and two receive sets (ids [world*cap],
    payload [world*cap*P]) used on alternate stages."""

    def __init__(self, cap: int, payload_row_bytes: int = 0, group=None, device=None):
        import ctypes
        from . import lib, _abi
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.cap, self.P = int(cap), int(payload_row_bytes)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        W = self.world
        sizes = {"counts": 8 * W, "done": 8 * W,
                 "ids0": 8 * W * self.cap, "ids1": 8 * W * self.cap}
        if self.P:
            sizes.update(pay0=W * self.cap * self.P, pay1=W * self.cap * self.P)
        self._own = {}
        for k, b in sizes.items():
            p = ctypes.c_void_p()
            _abi.call("hs_ipc_alloc", max(int(b), 16), ctypes.byref(p))
            self._own[k] = int(p.value)
        handles = {}
        for k, p in self._own.items():
            h = ctypes.create_string_buffer(64)
            if W > 1:
                _abi.call("hs_ipc_handle", p, h)
            handles[k] = bytes(h.raw)
        allh = [None] * W
        if W > 1:
            dist.all_gather_object(allh, handles, group=group)
        else:
            allh = [handles]
        self._opened = []
        self.peer = {k: [0] * W for k in self._own}
        for h in range(W):
            for k in self._own:
                if h == self.rank:
                    self.peer[k][h] = self._own[k]
                else:
                    p = ctypes.c_void_p()
                    hb = ctypes.create_string_buffer(allh[h][k], 64)
                    _abi.call("hs_ipc_open", hb, ctypes.byref(p))
                    self.peer[k][h] = int(p.value)
                    self._opened.append(int(p.value))
        self.ws = torch.zeros(256, dtype=torch.uint8, device=self.device)
        self.recv_count = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)   # STATUS_TIMEOUT
        self.epoch = 0
        self._lib = lib

    def recv_ids(self, parity: int) -> torch.Tensor:
        return torch.as_tensor(_DevArray(self._own[f"ids{parity}"], (self.world * self.cap,), "<i8"),
                               device=self.device)

    def recv_payload(self, parity: int) -> torch.Tensor | None:
        if not self.P:
            return None
        return torch.as_tensor(_DevArray(self._own[f"pay{parity}"], (self.world * self.cap, self.P), "|u1"),
                               device=self.device)

    def forward(self, ids: torch.Tensor, count: torch.Tensor, *, dest_ranks: list[int] | None = None,
                payload: torch.Tensor | None = None, stream=None):
        """Forward this rank's compacted deferred list ``ids[:count]`` (``count``:
        device int64[1], e.g. d_counts[1:2]).  Returns (recv_ids, recv_payload,
        recv_count) -- device tensors of this forward's receive set (alternating),
        recv_count a device int64[1]; nothing is read back to the host."""
        from . import forward_publish, forward_scatter, forward_wait
        self.epoch += 1
        par = self.epoch & 1
        dest = list(range(self.world)) if dest_ranks is None else list(dest_ranks)
        forward_publish(count, self.cap, self.rank, self.peer["counts"], self.epoch, stream=stream)
        forward_scatter(ids, self.cap, self.rank, self._own["counts"], self.peer["done"],
                        self.peer[f"ids{par}"], dest, self.epoch, self.recv_count, self.ws,
                        payload=payload, payload_row_bytes=self.P if payload is not None else 0,
                        peer_recv_payload=self.peer.get(f"pay{par}"), status=self.status,
                        stream=stream)
        forward_wait(self._own["done"], self.world, self.epoch, status=self.status, stream=stream)
        return self.recv_ids(par), self.recv_payload(par), self.recv_count

    def close(self):
        from . import _abi
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            _abi.call("hs_ipc_close", p)
        for p in self._own.values():
            _abi.call("hs_ipc_free", p)
        self._opened, self._own = [], {}
