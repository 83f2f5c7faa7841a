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


def replica_counts(world: int, reach: list[float], cost: list[float]) -> list[int]:
    """Replicas per model for the PLACED placement, from the
    zero-queuing rule of P:627-640 (§V-C): R_m S_m proportional to rho_m l_m
    ("the replications (R_1..R_n) should be (rho_1 l_1, .., rho_n l_n)/R_m ...
    round the real number to the nearest positive integer"), with
    rho_m the fraction of requests reaching model m, l_m its per-request cost
    and S_m = 1 (no model partitioning).  The world's GPUs are shared out:
    R_m = max(1, round(world * rho_m l_m / sum_j rho_j l_j)), then trimmed
    (largest first) or topped up (largest remainder first) until sum R_m ==
    world when the models fit, else each model keeps one replica."""
    w = [max(0.0, float(r)) * max(0.0, float(c)) for r, c in zip(reach, cost)]
    K = len(w)
    tot = sum(w)
    if tot <= 0:
        return [1] * K
    exact = [world * x / tot for x in w]
    R = [max(1, int(round(x))) for x in exact]
    if K > world:
        return [1] * K
    while sum(R) > world:
        i = max((i for i in range(K) if R[i] > 1), key=lambda i: R[i] - exact[i])
        R[i] -= 1
    while sum(R) < world:
        i = max(range(K), key=lambda i: exact[i] - R[i])
        R[i] += 1
    return R


def placed_ranks(world: int, replicas: list[int]) -> list[list[int]]:
    """Ranks hosting each model's replicas: consecutive blocks of the rank
    range, wrapping around (models share GPUs when sum R_m > world)."""
    out, start = [], 0
    for r in replicas:
        out.append([(start + i) % world for i in range(r)])
        start = (start + r) % world
    return out


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


class PeerGroup:
    """The multi-GPU group of the cascade over peer memory (hs_peer_t): one
    region per rank (hs_ipc_alloc), mapped into every rank's process with CUDA
    IPC -- handles exchanged once with ``all_gather_object`` over the process
    group -- so that the library's kernels forward deferred requests
    (hs_peer_forward, hs_cascade_step_peer) and sum the calibration histograms
    (hs_calibrate_thresholds_peer) through NVLink / NVSwitch with no host round
    trip and no NCCL on the data path.  ``cap``: the largest batch any rank
    routes in a stage; ``K``: stages (one receive count per forward)."""

    def __init__(self, cap: int, payload_row_bytes: int = 0, log2_bins: int = 12, K: int = 8,
                 group=None, device=None, *, _local=None):
        import ctypes
        from . import _abi, peer_region_bytes
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if _local is not None:                      # one process driving several ranks (tests)
            self.rank, self.world, regions = _local
            self._own, self._opened = None, []
        else:
            self.world = dist.get_world_size(group) if dist.is_initialized() else 1
            self.rank = dist.get_rank(group) if dist.is_initialized() else 0
            nbytes = peer_region_bytes(self.world, cap, payload_row_bytes, log2_bins)
            p = ctypes.c_void_p()
            _abi.call("hs_ipc_alloc", max(nbytes, 256), ctypes.byref(p))
            self._own = int(p.value)
            self._opened = []
            regions = [0] * self.world
            regions[self.rank] = self._own
            if self.world > 1:
                h = ctypes.create_string_buffer(64)
                _abi.call("hs_ipc_handle", self._own, h)
                allh = [None] * self.world
                dist.all_gather_object(allh, bytes(h.raw), group=group)
                for r in range(self.world):
                    if r == self.rank:
                        continue
                    q = ctypes.c_void_p()
                    _abi.call("hs_ipc_open", ctypes.create_string_buffer(allh[r], 64), ctypes.byref(q))
                    regions[r] = int(q.value)
                    self._opened.append(int(q.value))
        g = _abi.PeerGroup()
        g.rank, g.world, g.cap = self.rank, self.world, int(cap)
        g.payload_row_bytes, g.log2_bins = int(payload_row_bytes), int(log2_bins)
        for r in range(self.world):
            g.region[r] = regions[r]
        self.g = g
        self.cap, self.P, self.q = int(cap), int(payload_row_bytes), int(log2_bins)
        self.recv_count = torch.zeros(max(K - 1, 1), dtype=torch.int64, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)

    @classmethod
    def local_group(cls, world: int, cap: int, payload_row_bytes: int = 0, log2_bins: int = 12,
                    K: int = 8, device=None):
        """``world`` ranks driven by ONE process on one GPU (virtual ranks, for
        tests): the regions are plain allocations shared by pointer."""
        import ctypes
        from . import _abi, peer_region_bytes
        nbytes = peer_region_bytes(world, cap, payload_row_bytes, log2_bins)
        regions = []
        for _ in range(world):
            p = ctypes.c_void_p()
            _abi.call("hs_ipc_alloc", max(nbytes, 256), ctypes.byref(p))
            regions.append(int(p.value))
        ranks = [cls(cap, payload_row_bytes, log2_bins, K, device=device, _local=(r, world, regions))
                 for r in range(world)]
        ranks[0]._owned_local = regions
        return ranks

    def recv_ids(self, set_: int) -> torch.Tensor:
        from . import lib
        import ctypes
        ptr = lib().hs_peer_recv_ids(ctypes.byref(self.g), int(set_))
        return torch.as_tensor(_DevArray(ptr, (self.world * self.cap,), "<i8"), device=self.device)

    def recv_payload(self, set_: int):
        from . import lib
        import ctypes
        if not self.P:
            return None
        ptr = lib().hs_peer_recv_payload(ctypes.byref(self.g), int(set_))
        return torch.as_tensor(_DevArray(ptr, (self.world * self.cap, self.P), "|u1"), device=self.device)

    def forward(self, stage: int, ids: torch.Tensor, count: torch.Tensor, *, payload=None,
                dest_ranks=None, stream=None):
        """Forward this rank's deferred list ``ids[:count]`` after stage
        ``stage`` (receive set stage % 2).  Returns (recv_ids, recv_payload,
        recv_count) -- device tensors; nothing is read back to the host."""
        from . import peer_forward
        peer_forward(self.g, stage % 2, ids, count, self.recv_count[stage:stage + 1], payload=payload,
                     dest_ranks=dest_ranks, status=self.status, stream=stream)
        return self.recv_ids(stage % 2), self.recv_payload(stage % 2), self.recv_count[stage:stage + 1]

    def close(self):
        from . import _abi
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            _abi.call("hs_ipc_close", p)
        if self._own:
            _abi.call("hs_ipc_free", self._own)
        for p in getattr(self, "_owned_local", []):
            _abi.call("hs_ipc_free", p)
        self._opened, self._own, self._owned_local = [], None, []
