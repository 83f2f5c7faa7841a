"""The user-facing router: calibrate thresholds on a validation set, then route
batches through the cascade -- a sequence of C-ABI calls, nothing else.

One ``Router`` per GPU.  With a ``dist.PeerGroup`` (``peer=``) the validation
set and the request stream are sharded over the ranks and every exchange runs
inside the library over peer memory: the integer calibration histograms are
summed inside the calibration kernel (hs_calibrate_thresholds_peer), and the
deferred requests of every stage are forwarded to the next stage's ranks
(hs_cascade_step_peer) -- the whole calibrate + K-stage step is one CUDA graph
with no host round trip.  With a ``torch.distributed`` process group instead,
the histograms are summed with an all-reduce between ``hs_calibrate_histogram``
and ``hs_calibrate_select`` (order-independent count merging), or by the
library's own NCCL communicator (``native_comm``).
"""
from __future__ import annotations

import torch

import dataclasses

from . import (Cascade, StageSpec, _calib_out, calibrate_begin, calibrate_hist_view,
               calibrate_histogram, calibrate_select, calibrate_thresholds, calibrate_thresholds_comm,
               calibrate_thresholds_peer,
               calibrate_workspace, confidence, confidence_batched, cascade_step, fit_temperature,
               perf_graph, route_compact, threshold_replay)


class Router:
    def __init__(self, stages: list[StageSpec], n_cap: int, n_val: int, device, *,
                 log2_bins: int = 12, payload_row_bytes: int = 0, group=None,
                 native_comm: bool = False, peer=None):
        self.stages = stages
        self.K = len(stages)
        self.n_cap = int(n_cap)
        self.n_val = int(n_val)
        self.q = int(log2_bins)
        self.device = torch.device(device)
        self.group = group
        self.peer = peer
        self.next_ranks = None      # placed placement: destination ranks per forward
        dev = self.device
        K = self.K
        # validation confidences of all K stages: rows 0..K-2 are the calibration input
        self.vconf_all = torch.empty(K, self.n_val, dtype=torch.float32, device=dev)
        self.vconf = self.vconf_all[: K - 1]
        self.vconf_last = self.vconf_all[K - 1]
        self.vok = torch.empty(K, self.n_val, dtype=torch.uint8, device=dev)
        L = max(s.seq_len for s in stages)
        self.conf_ws = torch.empty(max(1, K * self.n_val * L * 5 + 1024), dtype=torch.uint8, device=dev)
        # one launch for every stage when the stages share a prediction shape
        s0 = stages[0]
        self.batched = K <= 8 and all((s.n_classes, s.seq_len, s.kind, s.reduce, s.top_k) ==
                                      (s0.n_classes, s0.seq_len, s0.kind, s0.reduce, 0)
                                      for s in stages)
        self.cal = _calib_out(K, dev, None)
        self.cal_ws = calibrate_workspace(K, self.q, dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.cascade = Cascade(self.n_cap, stages, dev, payload_row_bytes)
        self.cascade.status = self.status
        # native_comm: the calibration all-reduce runs inside the library on its
        # own NCCL communicator (hs_calibrate_thresholds_comm); the unique id is
        # shared once over the torch.distributed group
        self.hs_comm = None
        if native_comm:
            from . import comm_create, comm_unique_id
            import torch.distributed as dist
            world = dist.get_world_size(group) if group is not None else 1
            rank = dist.get_rank(group) if group is not None else 0
            uid = [comm_unique_id() if rank == 0 else None]
            if group is not None:
                dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0), group=group)
            self.hs_comm = comm_create(uid[0], rank, world, self.device.index or 0)

    # ---- offline: Alg. 1 / AP thresholds -----------------------
    def calibrate(self, val_logits: list, labels: torch.Tensor, *, target: int = -1,
                  time_val=None, stream=None) -> dict:
        """val_logits[k]: stage k's logits of the validation shard ([n_val*L, stride]);
        labels: int32 [n_val*L].  Thresholds stay on the device (self.cal['t']).
        ``time_val``: a pair of CUDA events recorded around the validation
        confidence launch(es)."""
        if time_val is not None:
            time_val[0].record()
        if self.batched:
            s = self.stages[0]
            confidence_batched(val_logits, [t.temperature for t in self.stages], n=self.n_val,
                               seq_len=s.seq_len, n_classes=s.n_classes, kind=s.kind,
                               reduce=s.reduce, labels=labels,
                               out={"conf": self.vconf_all.view(-1), "correct": self.vok.view(-1)},
                               want_argmax=False,
                               ws=self.conf_ws, status=self.status, stream=stream)
        else:
            for k, s in enumerate(self.stages):
                out = {"conf": self.vconf_all[k], "correct": self.vok[k]}
                confidence(val_logits[k], n=self.n_val, seq_len=s.seq_len, n_classes=s.n_classes,
                           temperature=s.temperature, kind=s.kind, reduce=s.reduce, labels=labels,
                           out=out, ws=self.conf_ws, status=self.status, top_k=s.top_k,
                           want_argmax=False, stream=stream)
        if time_val is not None:
            time_val[1].record()
        if self.peer is not None:
            calibrate_thresholds_peer(self.vconf, self.vok, self.peer.g, log2_bins=self.q, target=target,
                                      out=self.cal, ws=self.cal_ws, status=self.peer.status,
                                      stream=stream)
        elif self.hs_comm is not None:
            calibrate_thresholds_comm(self.vconf, self.vok, self.hs_comm, log2_bins=self.q,
                                      target=target, out=self.cal, ws=self.cal_ws, stream=stream)
        elif self.group is None:
            calibrate_thresholds(self.vconf, self.vok, log2_bins=self.q, target=target,
                                 out=self.cal, ws=self.cal_ws, stream=stream)
        else:
            import contextlib
            import torch.distributed as dist
            hist = calibrate_hist_view(self.cal_ws, self.q)
            # dist.all_reduce runs on torch's current stream: make it the
            # caller's, so histogram -> all-reduce -> select stay ordered
            ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
            with ctx:
                calibrate_begin(self.K, self.q, target, self.cal_ws)
                for k in range(self.K - 1):
                    calibrate_histogram(self.vconf, self.vok, k, self.cal["b"], log2_bins=self.q,
                                        ws=self.cal_ws)
                    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=self.group)
                    calibrate_select(self.K, k, self.cal, log2_bins=self.q, ws=self.cal_ws)
        return self.cal

    # ---- offline: temperature scaling (Eq. 1) ---------------------
    def fit_temperatures(self, val_logits: list, labels: torch.Tensor, *, t_lo: float | None = None,
                         t_hi: float | None = None, stream=None) -> list:
        """Fit one temperature per stage model on its validation logits (all
        models in one hs_fit_temperature launch; token rows of generation models
        are samples) and use them from now on (the confidence kernels take T as
        a host value, so this reads the K temperatures back: offline step)."""
        L = max(s.seq_len for s in self.stages)
        kw = {} if t_lo is None else {"t_lo": t_lo, "t_hi": t_hi}
        r = fit_temperature(val_logits, labels, n=self.n_val * L,
                            n_classes=self.stages[0].n_classes, stream=stream, **kw)
        temps = [float(t) for t in r["T"].cpu().tolist()]
        self.stages = [dataclasses.replace(s, temperature=t) for s, t in zip(self.stages, temps)]
        self.cascade.stages = self.stages
        self.temperature_fit = r
        return temps

    # ---- offline: threshold performance graph, AP / EO (Alg. 1) -------------
    def performance_graph(self, weights, *, log2_bins: int = 4, bvecs: torch.Tensor | None = None,
                          stream=None) -> dict:
        """Replay the cascade on the last calibrated validation confidences for
        every vector of the (B+2)^(K-1) grid (or ``bvecs``) with integer energy
        weights per model visit; returns the frontier, and the AP / EO vectors'
        threshold indices and thresholds (host lists)."""
        from . import grid_vector
        r = threshold_replay(self.vconf, self.vok, weights, log2_bins=log2_bins, bvecs=bvecs,
                             stream=stream)
        g = perf_graph(r["correct"], r["energy"], self.n_val, model_correct=r["model_correct"],
                       K=self.K, stream=stream)
        n = int(g["front_n"].item())
        pick = g["pick"].cpu().tolist()
        B = 1 << log2_bins

        def vec(s):
            if s < 0:
                return None
            b = grid_vector(s, self.K, log2_bins) if bvecs is None else bvecs[s].cpu().tolist()
            return {"b": b, "t": [float("inf") if x == B + 1 else x / B for x in b] + [0.0],
                    "correct": int(r["correct"][s]), "energy": int(r["energy"][s])}

        return {"front_c": g["front_c"][:n].cpu(), "front_e": g["front_e"][:n].cpu(),
                "front_s": g["front_s"][:n].cpu(), "ap": vec(pick[0]), "eo": vec(pick[1]),
                "replay": r}

    # ---- online: the cascade ------------------------------------
    def route(self, logits: list, *, n: int | None = None, ids=None, payload=None,
              by_id: bool = True, thresholds=None, overlap_first: bool = False, next_ranks=None,
              events=None, upto: int | None = None, split: bool = False, stream=None):
        """Route a batch; thresholds default to the calibrated device vector.
        ``overlap_first``: stage 1's confidence runs next to the calibration
        (HS_STEP_OVERLAP_PREVIOUS; it reads neither the calibration's buffers nor
        is read by it -- only the threshold test waits for the thresholds)."""
        thr = self.cal["t"] if thresholds is None else thresholds
        self.cascade.route(logits, thr, n=n, ids=ids, payload=payload, by_id=by_id,
                           overlap_first=overlap_first, peer=self.peer,
                           next_ranks=next_ranks if next_ranks is not None else self.next_ranks,
                           events=events, upto=upto, split=split, stream=stream)
        return self.cascade
