"""bench.py -- HybridServe cascade router on B200: requests routed/s and logits HBM GB/s.

One step = one pass of the whole hot path over one batch:
  (1) confidence of every stage model on the validation shard (K launches),
  (2) AP threshold calibration (histogram + select per round; NCCL all-reduce of
      the integer histograms when N > 1),
  (3) routing of the request batch through the K-stage cascade with the
      device-resident thresholds: per stage confidence -> threshold test ->
      stable compaction (+ gather).
Inputs are resident in HBM (per-stage logits indexed by request id, generated
by the seeded keyed generator before timing); the working set (~3 GB at C2) is
far larger than the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "requests routed/sec and logits HBM GB/s (% of peak) at 1/2/4/8 B200"
CONFIG_TEXT = {
    "c1": "2-stage ViT-S->ViT-L cascade, 4,096 requests x 1,000 classes fp32, calibrated on 4,096 validation samples",
    "c2": "5-stage ViT family cascade, 262,144 requests x 1,000 classes bf16 per GPU, thresholds calibrated on 50,000 validation samples",
    "c3": "4-size T5 cascade, 2,048 sequences x 64 tokens x 32,128 vocab bf16 per GPU (16,384 over 8 GPUs), MIN token confidence, 256 B payload gathered, 512 validation sequences per GPU",
    "c4": "3-stage Llama-like next-token cascade, 8,192 requests x 128,256 vocab bf16 per GPU, entropy confidence, 8 KB hidden-state payload gathered",
    "c5": "5-stage ViT streaming cascade, 1,048,576 requests x 1,000 classes bf16 per GPU (8M over 8 GPUs), validation 131,072 per GPU",
    "c5s": "5-stage ViT streaming cascade, STRONG scaling: 8,388,608 requests x 1,000 classes bf16 in total, "
           "2^23 / N per GPU (validation 2^20 / N per GPU)",
    "c5p": "5-stage ViT cascade, 16,384 requests x 1,000 classes bf16 per GPU, each request carrying its "
           "3 x 224 x 224 u8 image (150,528 B payload) that is gathered / forwarded with every deferral",
    "c3k": "c3 with the Top-K (K = 10) restricted token confidence of P:420-424 (NEXT-2), MIN over 64 tokens",
    "c3m": "c3 with the MEAN of the 64 token confidences as the sequence confidence (north_star; the paper's is MIN, P:423)",
    "c2skip": "NEXT-1: the C2 cascade (262,144 requests x 1,000 bf16, 5 ViT models, calibrated on 50,000) with "
              "skip connections -- a deferred request jumps to model k+1+j by the band of [0, t_k) its "
              "confidence falls in (uniform bands, P:497-541); logits indexed by request id; the plain "
              "cascade on the same logits is timed in the same run",
    "c2g": "NEXT-4: threshold performance graph of the 5 C2 ViT stage models: the exhaustive q = 4 grid (18^4 = 104,976 threshold vectors) replayed on the 50,000-sample validation set per GPU, Pareto frontier, AP and EO picks",
    "c2t": "NEXT-3: temperature fitting (Eq. 1, P:384-389) of the 5 C2 ViT stage models on the 50,000-sample validation set per GPU, 1,000 classes bf16, T in [e^-4, e^4]",
}
METRIC_TEMP = "temperature fitting (Eq. 1): stage-model validation rows fitted per second"
METRIC_GRAPH = "threshold performance graph (Alg. 1): threshold-vector x validation-sample cascade replays per second"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIG_TEXT))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="run routing stage 1 strictly after the calibration (no PDL overlap)")
    ap.add_argument("--split", action="store_true",
                    help="run each stage's compaction on a side stream next to the next stage's "
                         "confidence (hs_cascade_confidence + count / hs_cascade_compact); A/B on one "
                         "B200: 0.415 ms vs 0.396 ms per C2 step for the default single-stream step")
    ap.add_argument("--native-comm", action="store_true",
                    help="calibration all-reduce inside libhs on its own NCCL communicator "
                         "(hs_calibrate_thresholds_comm) instead of torch.distributed")
    ap.add_argument("--force-dist", action="store_true",
                    help="initialise NCCL even at one GPU (exercises the sharded calibration path)")
    ap.add_argument("--layout", default="dense", choices=["by_id", "dense"],
                    help="by_id: stage k's logits exist for every request id and the batch "
                         "gathers its rows; dense: stage k's logits are the dense batch of "
                         "the requests that reach model k, in order (the model ran on that "
                         "batch only, P:320-322)")
    ap.add_argument("--placement", default="balanced", choices=["balanced", "placed", "local", "nccl"],
                    help="balanced (default): after every stage the global stable deferred list is "
                         "re-spread in contiguous blocks over all ranks by the library's kernels over "
                         "peer memory (hs_cascade_step_peer; calibration histograms summed inside the "
                         "calibration kernel, hs_calibrate_thresholds_peer) -- one CUDA graph per "
                         "step, no host round trip; at one GPU the exchange is the identity. "
                         "placed: the same exchange, but stage k's batch goes only to the ranks holding "
                         "model k's replicas, R_m proportional to reach_m x cost_m (P:627-640). "
                         "local: every rank serves every stage of its own shard (replicas, no "
                         "exchange).  nccl: the balanced re-spread with torch.distributed NCCL "
                         "(count all-gather + all-to-all, host split sizes, eager) -- the baseline")
    ap.add_argument("--requests", type=int, default=0,
                    help="override the requests per GPU of the config (debugging / scaled runs; the "
                         "workload name then carries the count)")
    ap.add_argument("--plumbing-check", action="store_true",
                    help="CPU self-test of the multi-rank launcher (no GPU): every rank joins a gloo "
                         "group, exchanges a handle with all_gather_object and reduces with the "
                         "bench's max/sum helpers; rank 0 prints one JSON line")
    ap.add_argument("--share-gpu", action="store_true",
                    help="test mode: every rank uses cuda:0 (several processes time-slice one GPU; "
                         "plumbing over gloo) -- exercises the multi-process peer path on one GPU")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML sampled every ~5 ms in a thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def init_dist(args, force: bool = False):
    """One process per GPU (torchrun env).  torch.distributed is plumbing only
    (barriers, max-over-ranks timing, the one-time IPC handle exchange); the
    data path of the balanced placement runs in libhs over peer memory.
    --share-gpu: every rank on cuda:0 with gloo plumbing (test mode)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpu:
        local = 0
    if world > 1 and not args.share_gpu and torch.cuda.device_count() < world:
        raise SystemExit(f"bench: {world} ranks need {world} visible GPUs, found {torch.cuda.device_count()}")
    torch.cuda.set_device(local)
    if world > 1 or force:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _dist_tensor(x, dtype):
    """A tensor on the device the process group's backend reduces on."""
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    return torch.tensor(x, dtype=dtype, device=dev)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world: int):
    """Element-wise max over ranks of a float or a list of floats."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = _dist_tensor(x if isinstance(x, list) else [x], torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist() if isinstance(x, list) else float(t[0].item())


def sum_over_ranks(x, world: int):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = _dist_tensor(x, torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


# ---------------------------------------------------------------------------
# workload (per rank): weak scaling -- every rank routes its own shard
# ---------------------------------------------------------------------------
def family(config: str, world: int = 1):
    import dataclasses
    from workload import synth
    f = synth.FAMILIES.get(config)
    if config == "c5":      # per-GPU shard of the 8-GPU streaming config
        f = synth.scaled(f, n=1 << 20, n_val=1 << 17)
    if config == "c5s":     # strong scaling: the whole 2^23-request job split over the GPUs
        f = dataclasses.replace(synth.scaled(synth.FAMILIES["c5"], n=(1 << 23) // world,
                                             n_val=(1 << 20) // world), name="c5s_vit5_strong_bf16")
    if config == "c5p":     # the NVLink-roofline variant: a 3x224x224 u8 image forwarded with each request
        f = dataclasses.replace(synth.scaled(synth.FAMILIES["c5"], n=16384, n_val=1 << 17),
                                name="c5p_vit5_image_payload_bf16", payload_bytes=150528)
    if config == "c3k":     # NEXT-2: the T5 shard with Top-K token confidence
        import dataclasses
        f = dataclasses.replace(synth.scaled(synth.FAMILIES["c3"], n=2048, n_val=512),
                                name="c3k_t5x4_top10_bf16", top_k=10)
    if config == "c3":      # per-GPU shard of the 8-GPU T5 config
        f = synth.scaled(f, n=2048, n_val=512)
    if config == "c3m":     # the same shard, MEAN sequence confidence
        import dataclasses
        f = dataclasses.replace(synth.scaled(synth.FAMILIES["c3"], n=2048, n_val=512),
                                name="c3m_t5x4_mean_bf16", reduce=2)
    return f


def build_inputs(fam, rank: int, dev):
    import torch
    import workload
    from workload import synth
    tdt = torch.bfloat16 if fam.dtype == "bf16" else torch.float32
    K = fam.K
    id0 = rank * fam.n
    vid0 = synth.VAL_ID_BASE + rank * fam.n_val
    # route logits: stage k's model output for every request id of this shard (row = id - id0)
    route = []
    for k in range(K):
        x = torch.empty(fam.n * fam.L, fam.C, dtype=tdt, device=dev)
        workload.gpu_logits(x, fam, k, id_base=id0, n=fam.n)
        route.append(x)
    val = []
    for k in range(K):
        x = torch.empty(fam.n_val * fam.L, fam.C, dtype=tdt, device=dev)
        workload.gpu_logits(x, fam, k, id_base=vid0, n=fam.n_val)
        val.append(x)
    labels = torch.empty(fam.n_val * fam.L, dtype=torch.int32, device=dev)
    workload.gpu_labels(labels, fam, id_base=vid0, n=fam.n_val)
    payload = None
    if fam.payload_bytes:
        payload = torch.randint(0, 255, (fam.n, fam.payload_bytes), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    return route, val, labels, payload


def committed_traffic(config: str, name: str = "r02_k1_traffic.json"):
    """DRAM bytes per launch of the roofline kernel from the committed ncu
    capture (profiles/r02_k1_traffic.json, written by tools/ncu_summary.py
    traffic), when it was taken on this config; else None."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        rec = json.load(open(path))
    except (OSError, ValueError):
        return None
    return rec.get("dram_bytes_per_launch") if rec.get("config") == config else None


def dense_stage_logits(fam, router, route, val, labels, payload, rank, dev, ids0=None, next_ranks=None):
    """--layout dense: learn, stage by stage (untimed), which requests reach
    each model on this rank and generate stage k's logits (same keyed
    generator, so the same values per request) as the dense batch of exactly
    those requests in order -- what model m_k produces when it runs on its
    batch only.  With a peer group the batch of stage k >= 2 on this rank is
    the block it RECEIVED from the forward after stage k-1 (requests of any
    rank).  The cascade is deterministic, so every timed step routes the same
    batches (asserted after timing)."""
    import torch
    import workload
    router.calibrate(val, labels)
    tdt = torch.bfloat16 if fam.dtype == "bf16" else torch.float32
    out = [route[0]] + [None] * (fam.K - 1)
    peer = router.peer
    for k in range(1, fam.K):
        # stages 0..k-1 on the batches known so far (every rank in lockstep)
        router.route(out, n=fam.n, ids=ids0, payload=payload, by_id=False, upto=k - 1, next_ranks=next_ranks)
        torch.cuda.synchronize()
        if peer is not None:
            nk = int(peer.recv_count[k - 1].item())
            ids = peer.recv_ids((k - 1) % 2)[:nk].clone()
        else:
            nk = int(router.cascade.counts[k - 1][1].item())
            ids = router.cascade.outs[k - 1]["next_ids"][:nk].clone()
            if ids0 is None:
                ids += rank * fam.n
        # the live rows are a view of a capacity-sized buffer (what a graph-
        # captured model stage writes into), so the confidence kernel may read
        # dense rows before the live count is known (HS_STEP_LOGITS_CAPACITY);
        # exact-sized when the capacity buffers would exceed 40 GB (c5s)
        cap_rows = fam.n * fam.L
        eb = 2 if fam.dtype == "bf16" else 4
        full = peer is None and (fam.K - 1) * cap_rows * fam.C * eb <= (40 << 30)
        buf = torch.empty(cap_rows if full else max(nk, 1) * fam.L, fam.C, dtype=tdt, device=dev)
        x = buf[: max(nk, 1) * fam.L]
        if nk:
            workload.gpu_logits(x, fam, k, ids=ids, n=nk)
        out[k] = x
        route[k] = None                    # the full-population tensor is not needed
    router.route(out, n=fam.n, ids=ids0, payload=payload, by_id=False, next_ranks=next_ranks)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out, dense_signature(router, fam)


def dense_signature(router, fam):
    import torch
    counts = router.cascade.counts.cpu().tolist()
    batch = []
    if router.peer is not None:
        batch = [int(x) for x in router.peer.recv_count[: fam.K - 1].cpu().tolist()]
    else:
        batch = [int(c[1]) for c in counts[:-1]]
    return counts, batch


def make_router(fam, dev, group, native_comm: bool = False, peer=None, n_cap=None):
    import paper_2505_12566_b200 as hs
    from paper_2505_12566_b200.router import Router
    stages = [hs.StageSpec(fam.C, fam.temps[k], fam.L, fam.kind, fam.reduce, fam.top_k)
              for k in range(fam.K)]
    return Router(stages, n_cap or fam.n, fam.n_val, dev, log2_bins=fam.log2_bins,
                  payload_row_bytes=fam.payload_bytes, group=group, native_comm=native_comm, peer=peer)


def timing_event():
    """A timing event usable inside a captured CUDA graph (recorded as an
    external event node), so the dominant kernel is timed inside the step."""
    import torch
    try:
        return torch.cuda.Event(enable_timing=True, external=True)
    except TypeError:
        return torch.cuda.Event(enable_timing=True)


def run_ours(args, world, rank, local):
    """The step of every config but c2g / c2t: calibration + K-stage routing.
    world > 1 with the balanced placement: a dist.PeerGroup -- the calibration
    histograms are summed inside the calibration kernel and every stage's
    deferred list is forwarded to its global block over peer memory, all inside
    one CUDA graph (hs_calibrate_thresholds_peer, hs_cascade_step_peer)."""
    import torch
    import torch.distributed as dist
    import paper_2505_12566_b200 as hs
    from paper_2505_12566_b200 import dist as hsd

    dev = torch.device("cuda", local)
    fam = family(args.config, world)
    if args.requests:
        import dataclasses
        fam = dataclasses.replace(fam, n=args.requests, name=f"{fam.name}_n{args.requests}")
    group = dist.group.WORLD if dist.is_initialized() else None
    route, val, labels, payload = build_inputs(fam, rank, dev)
    peer = None
    placed = args.placement == "placed" and world > 1
    # placed: a rank holding a model's replica can receive up to world x its shard
    cap = fam.n * (world if placed else 1)
    if world > 1 and args.placement in ("balanced", "placed"):
        peer = hsd.PeerGroup(cap, fam.payload_bytes, fam.log2_bins, K=fam.K, group=group, device=dev)
    router = make_router(fam, dev, None if peer is not None else group, native_comm=args.native_comm,
                         peer=peer, n_cap=cap)
    next_ranks = None
    if placed:
        # replicas from the calibrated validation reach (global, summed inside the
        # calibration kernel) and per-visit costs (GRAPH_W: synthetic ViT ratios)
        router.calibrate(val, labels)
        reach = [float(x) for x in router.cal["reach"].cpu().tolist()]
        replicas = hsd.replica_counts(world, [r / max(reach[0], 1.0) for r in reach], list(GRAPH_W[:fam.K]))
        ranks = hsd.placed_ranks(world, replicas)
        next_ranks = ranks[1:]
        router.next_ranks = next_ranks
    ids0 = (torch.arange(rank * fam.n, (rank + 1) * fam.n, dtype=torch.int64, device=dev)
            if peer is not None else None)
    ev = (timing_event(), timing_event())
    dense = args.layout == "dense"
    if peer is not None and not dense:
        raise SystemExit("bench: the balanced placement routes dense stage batches (--layout dense)")
    if dense:
        route, dense_sig = dense_stage_logits(fam, router, route, val, labels, payload, rank, dev, ids0,
                                              next_ranks=next_ranks)
    K = fam.K
    sev = [timing_event() for _ in range(2 * K)] + [timing_event()]

    def step(events=None):
        # K1 on the validation shard is the timed launch (events around it); the
        # routing stage-1 K1 then runs next to the latency-bound calibration
        router.calibrate(val, labels, time_val=ev)
        router.route(route, n=fam.n, ids=ids0, payload=payload, overlap_first=not args.no_overlap,
                     by_id=not dense, events=events, split=dense and peer is None and args.split,
                     next_ranks=next_ranks)
        if events is not None:
            sev[2 * K].record()

    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    torch.cuda.synchronize()
    use_graph = not args.no_graph
    graph = None
    launches_per_step = None
    if use_graph:
        try:
            l0 = hs.launch_count()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
            launches_per_step = hs.launch_count() - l0
            graph.replay()
            torch.cuda.synchronize()
        except Exception as e:  # collectives that cannot be captured: eager timing
            print(f"[bench] graph capture failed ({e}); timing eagerly", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    l_before = hs.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    k_ms = []
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            t0.record(stream)
            for _ in range(args.steps):
                if graph is not None:
                    graph.replay()
                else:
                    step()
            t1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    total_ms = t0.elapsed_time(t1)
    clocks = clk.summary()
    gpu_launches = (launches_per_step * args.steps) if graph is not None else (hs.launch_count() - l_before)
    # per-launch duration of the dominant kernel: one more timed pass, recording each step's events
    k_ms, s_ms = [], []
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for _ in range(min(args.steps, 50)):
            s0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            s1.record(stream)
            stream.synchronize()
            k_ms.append(ev[0].elapsed_time(ev[1]))
            s_ms.append(s0.elapsed_time(s1))
    kernel_ms = sum(k_ms) / len(k_ms)
    s_ms.sort()
    step_pct = {"p10": s_ms[len(s_ms) // 10], "p50": s_ms[len(s_ms) // 2],
                "p90": s_ms[(9 * len(s_ms)) // 10], "n": len(s_ms),
                "note": "per-step CUDA-event times of a second, individually synchronised pass"}
    ms = max_over_ranks(total_ms, world) / args.steps
    # per-stage breakdown (an eager, event-instrumented pass: the forward is
    # launched as its own call between the events), max over ranks
    barrier(world)
    with torch.cuda.stream(stream):
        for _ in range(3):
            step(events=sev)
        stream.synchronize()
    stage_ms = [sev[2 * k].elapsed_time(sev[2 * k + 1]) for k in range(K)]
    fwd_ms = [sev[2 * k + 1].elapsed_time(sev[2 * k + 2]) for k in range(K - 1)]
    stage_ms = max_over_ranks(stage_ms, world)
    fwd_ms = max_over_ranks(fwd_ms, world) if K > 1 else []
    # cascade statistics (identical every step): reach per stage (summed over ranks)
    if dense:
        assert dense_signature(router, fam) == dense_sig, "dense layout: the cascade changed between steps"
    counts = router.cascade.counts.cpu().tolist()
    if peer is not None:
        batch_local = [fam.n] + [int(x) for x in peer.recv_count[: K - 1].cpu().tolist()]
    else:
        batch_local = [fam.n] + [c[1] for c in counts[:-1]]
    deferred_local = [c[1] for c in counts[:-1]]
    reach = [int(x) for x in sum_over_ranks([float(b) for b in batch_local], world)]
    st = int(router.status.item()) | (int(peer.status.item()) if peer is not None else 0)
    # algorithmic bytes of one step (logits dominate): validation sweep + routing of each stage batch
    row_b = fam.row_bytes
    val_bytes = K * fam.n_val * row_b
    step_bytes = val_bytes + sum(batch_local) * row_b
    step_bytes_all = sum_over_ranks([float(step_bytes)], world)[0]
    n_all = fam.n * world
    value = n_all / (ms / 1e3)
    peak, peak_src = peaks()
    # dominant kernel: K1 over the validation shard, all K stages in one launch:
    # per item, its L token rows of logits (row_b) + per token conf (4 B),
    # label (4 B) and correct bit (1 B) (the validation argmax is not stored)
    k_bytes = K * fam.n_val * (row_b + 9 * fam.L)
    achieved = k_bytes / (kernel_ms / 1e3) / 1e9
    traffic = committed_traffic(args.config)
    e2e = (run_e2e(args, fam, router, route, val, labels, payload, stream, world, ids0)
           if args.e2e_steps > 0 else None)
    line = {
        "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if args.config == "c5s" else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": fam.name, "description": CONFIG_TEXT[args.config],
                   "requests_per_gpu": fam.n, "validation_per_gpu": fam.n_val, "K": K,
                   "classes": fam.C, "seq_len": fam.L, "logits_dtype": fam.dtype,
                   "confidence": ["maxprob", "maxprob_sq", "entropy"][fam.kind]
                   + (f" over the top {fam.top_k} logits" if fam.top_k else ""),
                   "sequence_reduce": ["none", "min", "mean"][fam.reduce],
                   "log2_bins": fam.log2_bins,
                   "parallelism": f"request-sharded dp{world}"
                   + (f", {'placed' if placed else 'balanced'} forwarding + calibration exchange over "
                      "peer memory (hs_peer_*)" if peer is not None else ", replicas (no exchange)"
                      if world > 1 else ""),
                   "placement": args.placement if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (per-step logits working set >> 126 MB)",
                   "logits_layout": args.layout,
                   "cuda_graph": graph is not None},
        "logits_GBps": step_bytes_all / (ms / 1e3) / 1e9,
        "logits_frac_of_peak": step_bytes_all / world / (ms / 1e3) / 1e9 / peak,
        "reach": reach, "thresholds": router.cal["t"].cpu().tolist(), "status": st,
        "stage_ms_max_over_ranks": stage_ms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ("conf_topk_kernel" if fam.top_k else
                                "conf_async_kernel" if fam.C * fam.elt_bytes <= 2048 else
                                "conf_warp_kernel" if fam.C * fam.elt_bytes <= 8192 else "conf_stream_kernel")
                     + f" (K1 on the validation shard: {K} stages x {fam.n_val} items in one launch"
                     + (", + K2 sequence reduce" if fam.L > 1 else "") + ")",
                     "bytes_per_launch": k_bytes, "avg_launch_ms": kernel_ms,
                     "peak_source": peak_src},
        "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clocks,
        "gpu_launches_per_step": gpu_launches / args.steps,
        "step_ms_percentiles": step_pct,
    }
    if fam.payload_bytes:
        # deferred requests carry their payload rows: gathered (read + write) at
        # every deferral on a single GPU, forwarded over NVLink at N > 1
        moved = sum_over_ranks([float(sum(deferred_local) * 2 * fam.payload_bytes)], world)[0]
        line["payload"] = {"row_bytes": fam.payload_bytes, "bytes_moved_per_step": moved,
                           "GBps_step": moved / (ms / 1e3) / 1e9,
                           "note": "gather K4 / peer scatter of the deferred rows; step-level rate"}
    if placed:
        line["config"]["replicas_per_model"] = replicas
        line["config"]["model_ranks"] = ranks
    if peer is not None:
        # forwarded ids (+ payload rows) per stage, NVLink bytes sent per rank
        fwd_items = [int(x) for x in sum_over_ranks([float(d) for d in deferred_local], world)]
        per_rank_bytes = max_over_ranks([float(d * (8 + fam.payload_bytes)) for d in deferred_local], world)
        line["comm"] = {
            "kind": "peer memory (CUDA IPC mappings; hs_peer_forward + in-kernel histogram exchange)",
            "world": world, "forwarded_items_per_stage": fwd_items,
            "bytes_sent_per_rank_max": per_rank_bytes,
            "forward_ms_max_over_ranks": fwd_ms,
            "nvlink_GBps_per_rank": [b / (t / 1e3) / 1e9 if t > 0 else None
                                     for b, t in zip(per_rank_bytes, fwd_ms)],
            "nvlink_peak_GBps_per_direction": 900.0,
            "note": "ids-only forwarding is latency-bound (flag round trip ~ us); the fraction of "
                    "NVLink peak is reported, not targeted"}
    return line, fam, route, val, labels, router
def run_nccl(args, world, rank, local):
    """Request-sharded cascade with the BALANCED placement done by
    torch.distributed NCCL -- the baseline of the peer-memory path: after
    every stage the global stable deferred list is re-spread in contiguous blocks
    over all ranks (count all-gather + one NCCL all-to-all of ids and payload),
    and each rank routes the block it received.  Calibration sums the per-rank
    histograms with an NCCL all-reduce.  Host round trip per stage (NCCL split
    sizes are host values), so the step runs eagerly (no CUDA graph)."""
    import torch
    import torch.distributed as dist
    import workload
    import paper_2505_12566_b200 as hs
    from paper_2505_12566_b200 import dist as hsd
    from workload import synth

    dev = torch.device("cuda", local)
    fam = family(args.config)
    K, n, P = fam.K, fam.n, fam.payload_bytes
    tdt = torch.bfloat16 if fam.dtype == "bf16" else torch.float32
    # stage 1: this rank's shard (global ids rank*n ..); later stages: any id of
    # the job can arrive here, so stage k >= 2 logits cover all world*n ids
    logits = []
    for k in range(K):
        rows = n if k == 0 else world * n
        x = torch.empty(rows * fam.L, fam.C, dtype=tdt, device=dev)
        workload.gpu_logits(x, fam, k, id_base=rank * n if k == 0 else 0, n=rows)
        logits.append(x)
    _, val, labels, payload = build_inputs(synth.scaled(fam, n=1), rank, dev)
    router = make_router(fam, dev, dist.group.WORLD)
    cap = world * n                          # worst case: everything lands on one rank
    ws = hs.workspace(hs.lib().hs_cascade_step_workspace(cap, fam.L), dev)
    ids0 = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int64, device=dev)
    pay0 = (torch.randint(0, 255, (n, P), dtype=torch.uint8, device=dev) if P else None)
    outs = [{"acc_ids": torch.empty(cap, dtype=torch.int64, device=dev),
             "acc_conf": torch.empty(cap, dtype=torch.float32, device=dev),
             "acc_pred": torch.empty(cap * fam.L, dtype=torch.int32, device=dev),
             "next_ids": torch.empty(cap, dtype=torch.int64, device=dev),
             "counts": torch.zeros(2, dtype=torch.int64, device=dev)} for _ in range(K)]
    if P:
        for o in outs:
            o["next_payload"] = torch.empty(cap * P, dtype=torch.uint8, device=dev)

    def step():
        cal = router.calibrate(val, labels)
        ids, pay, nb = ids0, pay0, n
        for k in range(K):
            row_index = ids - rank * n if k == 0 else ids
            o = outs[k]
            hs.cascade_step(k, K, logits[k], cal["t"][k:k + 1], n=nb, seq_len=fam.L,
                            n_classes=fam.C, temperature=fam.temps[k], kind=fam.kind,
                            reduce=fam.reduce, row_index=row_index, ids=ids, payload=pay,
                            payload_row_bytes=P, out=o, ws=ws)
            if k == K - 1:
                break
            nids, npay, nb = hsd.forward_deferred(
                o["next_ids"], o["counts"][1:2],
                payload=o["next_payload"][: cap * P].view(cap, P) if P else None)
            ids, pay = nids, npay

    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    l0 = hs.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = max_over_ranks(t0.elapsed_time(t1), world) / args.steps
    launches = hs.launch_count() - l0
    value = world * n / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": fam.name, "description": CONFIG_TEXT[args.config],
                   "requests_per_gpu": n, "validation_per_gpu": fam.n_val, "K": K,
                   "classes": fam.C, "seq_len": fam.L, "logits_dtype": fam.dtype,
                   "parallelism": f"request-sharded dp{world}, balanced all-to-all forwarding "
                                  "(torch.distributed NCCL, host split sizes, eager)",
                   "l2": "inputs larger than L2", "cuda_graph": False},
        "gpu_launches": launches, "clocks": clk.summary(), "e2e": None,
        "thresholds": router.cal["t"].cpu().tolist(),
    }
    return line, fam


def run_e2e(args, fam, router, route, val, labels, payload, stream, world, ids0=None):
    """Same metric through the public API from pinned HOST buffers: every step copies
    its inputs host->device and reads the per-request results back."""
    import torch
    steps = args.e2e_steps
    in_bytes = sum(x.numel() * x.element_size() for x in list(route) + list(val) if x is not None)
    if in_bytes > (8 << 30):   # pinned host copies of > 8 GB per rank: not run (c5s at few GPUs)
        return {"skipped": f"{in_bytes / 1e9:.1f} GB of inputs per step per rank exceed the 8 GB "
                           "pinned-host budget of the e2e leg"}
    host_route = [x.cpu().pin_memory() for x in route]
    host_val = [x.cpu().pin_memory() for x in val]
    host_lab = labels.cpu().pin_memory()
    host_pay = payload.cpu().pin_memory() if payload is not None else None
    outs = router.cascade.outs
    res_host = [torch.empty(fam.n * 8, dtype=torch.uint8).pin_memory() for _ in outs]
    cnt_host = torch.empty(fam.K, 2, dtype=torch.int64).pin_memory()
    h2d = sum(x.numel() * x.element_size() for x in host_route + host_val) + \
        host_lab.numel() * 4 + (host_pay.numel() if host_pay is not None else 0)
    d2h = 0

    def once():
        nonlocal d2h
        for d, h in zip(route, host_route):
            d.copy_(h, non_blocking=True)
        for d, h in zip(val, host_val):
            d.copy_(h, non_blocking=True)
        labels.copy_(host_lab, non_blocking=True)
        if payload is not None:
            payload.copy_(host_pay, non_blocking=True)
        router.calibrate(val, labels)
        router.route(route, n=fam.n, ids=ids0, payload=payload, by_id=args.layout != "dense")
        cnt_host.copy_(router.cascade.counts, non_blocking=True)
        # accepted ids of every stage (the answers' request ids)
        for o, h in zip(outs, res_host):
            h.view(torch.int64).copy_(o["acc_ids"], non_blocking=True)
        d2h = cnt_host.numel() * 8 + sum(h.numel() for h in res_host)

    with torch.cuda.stream(stream):
        once()
    torch.cuda.synchronize()
    barrier(world)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        t0.record(stream)
        for _ in range(steps):
            once()
        t1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(t0.elapsed_time(t1), world) / steps
    return {"value": fam.n * world / (ms / 1e3), "unit": "requests/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "steps": steps}


# ---------------------------------------------------------------------------
# NEXT-1: skip connections (--config c2skip)
# ---------------------------------------------------------------------------
def run_skip(args, world, rank, local):
    """Step = calibration + routing through the SKIP cascade (hs_skip_select /
    hs_confidence / hs_skip_route per model; uniform bands); the plain
    cascade (by-id layout) on the same logits and thresholds is timed in the
    same run for the comparison the paper draws (tail latency).  N > 1:
    independent replicas on shard-local requests."""
    import torch
    import paper_2505_12566_b200 as hs
    dev = torch.device("cuda", local)
    fam = family("c2")
    route, val, labels, _ = build_inputs(fam, rank, dev)
    router = make_router(fam, dev, None)
    stages = [hs.StageSpec(fam.C, fam.temps[k]) for k in range(fam.K)]
    sc = hs.SkipCascade(fam.n, stages, dev, mode=hs.SKIP_UNIFORM)

    def step_skip():
        router.calibrate(val, labels)
        sc.route(route, router.cal["t"])

    def step_plain():
        router.calibrate(val, labels)
        router.route(route, by_id=True, overlap_first=not args.no_overlap)

    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    graphs = {}
    for name, fn in (("skip", step_skip), ("plain", step_plain)):
        with torch.cuda.stream(stream):
            for _ in range(max(args.warmup, 3)):
                fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        l0 = hs.launch_count()
        with torch.cuda.graph(g, stream=stream):
            fn()
        graphs[name] = (g, hs.launch_count() - l0)
        g.replay()
        torch.cuda.synchronize()
    times = {}
    barrier(world)
    with ClockSampler(local) as clk:
        for name in ("skip", "plain", "skip"):
            g = graphs[name][0]
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                t0.record(stream)
                for _ in range(args.steps):
                    g.replay()
                t1.record(stream)
            torch.cuda.synchronize()
            times[name] = t0.elapsed_time(t1) / args.steps      # skip: the second pass
    ms = max_over_ranks(times["skip"], world)
    ms_plain = max_over_ranks(times["plain"], world)
    sel = sc.sel_counts.cpu().tolist()
    visits_skip = [fam.n] + [int(c[1]) for c in sel[1:]]
    counts = router.cascade.counts.cpu().tolist()
    visits_plain = [fam.n] + [int(c[1]) for c in counts[:-1]]
    answered_skip = [int(c[0]) for c in sc.counts.cpu().tolist()]
    line = {
        "metric": METRIC, "value": fam.n * world / (ms / 1e3), "unit": "requests/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "c2skip_vit5_uniform_bands", "description": CONFIG_TEXT["c2skip"],
                   "requests_per_gpu": fam.n, "validation_per_gpu": fam.n_val, "K": fam.K,
                   "classes": fam.C, "logits_dtype": fam.dtype, "logits_layout": "by_id",
                   "parallelism": f"independent replicas x{world}",
                   "l2": "inputs larger than L2", "cuda_graph": True},
        "thresholds": router.cal["t"].cpu().tolist(),
        "model_visits_skip": visits_skip, "answered_per_model_skip": answered_skip,
        "model_visits_plain": visits_plain,
        "plain_cascade_ms_per_step": ms_plain,
        "skip_vs_plain_logits_bytes": sum(visits_skip) / max(sum(visits_plain), 1),
        "gpu_launches": graphs["skip"][1] * args.steps, "gpu_launches_per_step": graphs["skip"][1],
        "clocks": clk.summary(), "e2e": None,
    }
    return line


# ---------------------------------------------------------------------------
# NEXT-3: temperature fitting on the validation set (--config c2t)
# ---------------------------------------------------------------------------
def run_temperature(args, world, rank, local):
    """Step = hs_fit_temperature over the validation shard of every stage model
    (one persistent launch: a max/label sweep + the Newton sweeps).  N > 1:
    independent replicas (each rank fits on its own shard; no collective)."""
    import torch
    import paper_2505_12566_b200 as hs
    dev = torch.device("cuda", local)
    fam = family("c2")
    _, val, labels, _ = build_inputs(synth_scaled(fam, n=1), rank, dev)
    K, n = fam.K, fam.n_val
    ws = torch.empty(hs.lib().hs_fit_temperature_workspace(K, n), dtype=torch.uint8, device=dev)
    out = {"T": torch.empty(K, dtype=torch.float32, device=dev),
           "nll": torch.empty(K, dtype=torch.float64, device=dev),
           "passes": torch.empty(K, dtype=torch.int32, device=dev),
           "used": torch.empty(K, dtype=torch.int64, device=dev)}
    status = torch.zeros(1, dtype=torch.int32, device=dev)

    def step():
        hs.fit_temperature(val, labels, out=out, ws=ws, status=status)

    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    torch.cuda.synchronize()
    graph = None
    launches_per_step = 1
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            l0 = hs.launch_count()
            step()
            launches_per_step = hs.launch_count() - l0
        graph.replay()
        torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            t0.record(stream)
            for _ in range(args.steps):
                graph.replay() if graph is not None else step()
            t1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(t0.elapsed_time(t1), world) / args.steps
    passes = out["passes"].cpu().tolist()
    T = out["T"].cpu().tolist()
    row_b = fam.row_bytes
    # algorithmic bytes of one launch: every sweep reads the rows of each model
    # still fitting (sweep 0 also reads the label and writes 8 B of row state;
    # later sweeps read it back)
    # rows of <= 2 KB fold the max/label sweep into the first Newton sweep, and
    # (n >= 32,768) start from <= 2 Newton sweeps over a 1/16 row sample
    sweep0 = 0 if row_b <= 2048 else 1
    sub = 2 * ((n + 15) // 16) * (row_b + 4) if (row_b <= 2048 and n >= 32768) else 0
    k_bytes = sum((sweep0 + p) * n * row_b + n * (4 + 8) + p * n * 8 + sub for p in passes)
    peak, peak_src = peaks()
    achieved = k_bytes / (ms / 1e3) / 1e9
    e2e = None
    if args.e2e_steps > 0:
        host_val = [x.cpu().pin_memory() for x in val]
        host_lab = labels.cpu().pin_memory()
        host_T = torch.empty(K, dtype=torch.float32).pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in host_val) + host_lab.numel() * 4

        def once():
            for d, h in zip(val, host_val):
                d.copy_(h, non_blocking=True)
            labels.copy_(host_lab, non_blocking=True)
            step()
            host_T.copy_(out["T"], non_blocking=True)

        with torch.cuda.stream(stream):
            once()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.e2e_steps):
                once()
            e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1), world) / args.e2e_steps
        e2e = {"value": K * n * world / (ems / 1e3), "unit": "rows/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": K * 4, "ms_per_step": ems, "steps": args.e2e_steps}
    line = {
        "metric": METRIC_TEMP, "value": K * n * world / (ms / 1e3), "unit": "rows/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "c2t_vit5_validation_temperature", "description": CONFIG_TEXT["c2t"],
                   "validation_per_gpu": n, "K": K, "classes": fam.C, "logits_dtype": fam.dtype,
                   "parallelism": f"independent replicas x{world} (shard-local fit)",
                   "l2": "inputs larger than L2 (500 MB of validation logits per sweep)",
                   "cuda_graph": graph is not None},
        "temperatures": T, "passes": passes, "status": int(status.item()),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": committed_traffic("c2t", "r01_tf_traffic.json"),
                     "kernel": "temp_fit_kernel (the whole step: one persistent cooperative launch; "
                               "full sweeps per model = passes, plus 2 warm-start sweeps over 1/16 "
                               "of the rows counted as an upper bound)",
                     "bytes_per_launch": k_bytes, "avg_launch_ms": ms, "peak_source": peak_src},
        "e2e": e2e, "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
        "gpu_launches_per_step": launches_per_step,
    }
    return line, fam, val, labels


GRAPH_Q = 4
GRAPH_W = (1, 2, 4, 8, 16)     # integer energy per visit, ViT-XS .. ViT-L (synthetic ratios)


def graph_inputs(fam, rank, dev):
    """The validation confidences / correct bits of every stage model (the input
    of Alg. 1), computed once on the GPU before timing."""
    import paper_2505_12566_b200 as hs
    _, val, labels, _ = build_inputs(synth_scaled(fam, n=1), rank, dev)
    r = hs.confidence_batched(val, fam.temps, labels=labels)
    K, n = fam.K, fam.n_val
    conf = r["conf"].view(K, n)[: K - 1].contiguous()
    ok = r["correct"].view(K, n).contiguous()
    return conf, ok


def run_graph(args, world, rank, local):
    """Step = hs_threshold_replay over the whole q = 4 grid + hs_perf_graph
    (frontier, AP, EO).  N > 1: independent replicas on shard-local samples."""
    import torch
    import paper_2505_12566_b200 as hs
    dev = torch.device("cuda", local)
    fam = family("c2")
    conf, ok = graph_inputs(fam, rank, dev)
    K, n = fam.K, fam.n_val
    S = hs.grid_size(K, GRAPH_Q)
    rws = torch.empty(hs.lib().hs_threshold_replay_workspace(K, n, GRAPH_Q), dtype=torch.uint8, device=dev)
    gws = torch.empty(hs.lib().hs_perf_graph_workspace(n), dtype=torch.uint8, device=dev)
    rout, gout = {}, {}

    def step():
        r = hs.threshold_replay(conf, ok, GRAPH_W, log2_bins=GRAPH_Q, out=rout, ws=rws)
        rout.update(r)
        g = hs.perf_graph(r["correct"], r["energy"], n, model_correct=r["model_correct"], K=K,
                          out=gout, ws=gws)
        gout.update(g)

    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    torch.cuda.synchronize()
    graph = None
    launches_per_step = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            l0 = hs.launch_count()
            step()
            launches_per_step = hs.launch_count() - l0
        graph.replay()
        torch.cuda.synchronize()
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    l_before = hs.launch_count()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            t0.record(stream)
            for _ in range(args.steps):
                graph.replay() if graph is not None else step()
            t1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(t0.elapsed_time(t1), world) / args.steps
    if launches_per_step is None:
        launches_per_step = (hs.launch_count() - l_before) / args.steps
    # the replay kernel alone (eager, CUDA events on its stream)
    rk = []
    with torch.cuda.stream(stream):
        for _ in range(10):
            ev[0].record(stream)
            hs.threshold_replay(conf, ok, GRAPH_W, log2_bins=GRAPH_Q, out=rout, ws=rws)
            ev[1].record(stream)
            stream.synchronize()
            rk.append(ev[0].elapsed_time(ev[1]))
    replay_ms = sorted(rk)[len(rk) // 2]
    evals = S * n
    # the exhaustive grid runs through the prefix histograms (q <= 5): one visit
    # per (prefix b_0..b_{K-3}, sample); its ALU work per visit is K-2 compares +
    # K-2 selects (answering model), 2 (correct bit), 2(K-2) (reach counts) and
    # 4 (histogram address + 64-bit add) thread instructions
    R = (1 << GRAPH_Q) + 2
    visits = (S // R) * n
    ops_per_visit = 4 * (K - 2) + 6
    clocks = clk.summary()
    mhz = clocks.get("sm_max_mhz") or 1965
    # the compares / selects / shifts / integer adds all issue to the ALU pipe:
    # reciprocal throughput 2 cycles per warp instruction per SMSP (B300_MICROARCH.md
    # "fma vs alu split", same SM design) = 16 lanes/clk/SMSP, 64/clk/SM
    peak = 148 * 4 * 16 * mhz * 1e6 / 1e12
    achieved = ops_per_visit * visits / (replay_ms / 1e3) / 1e12
    pick = gout["pick"].cpu().tolist()
    fn = int(gout["front_n"].item())
    line = {
        "metric": METRIC_GRAPH, "value": evals * world / (ms / 1e3), "unit": "replays/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": "c2g_vit5_grid_q4", "description": CONFIG_TEXT["c2g"],
                   "validation_per_gpu": n, "K": K, "log2_bins": GRAPH_Q, "vectors": S,
                   "energy_weights": list(GRAPH_W),
                   "parallelism": f"independent replicas x{world} (shard-local graph)",
                   "l2": "samples re-read from L2 by every CTA (2.5 MB working set, by design)",
                   "cuda_graph": graph is not None},
        "frontier_points": fn, "ap_vector": hs.grid_vector(pick[0], K, GRAPH_Q) if pick[0] >= 0 else None,
        "eo_vector": hs.grid_vector(pick[1], K, GRAPH_Q) if pick[1] >= 0 else None,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tinstr/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": f"hs_threshold_replay: replay_hist_kernel<{K - 1}> + prep / finish "
                               f"({S // R} prefixes x {n} samples = {visits} visits, {ops_per_visit} "
                               "algorithmic ALU instructions per visit; timed as the whole call)",
                     "avg_launch_ms": replay_ms,
                     "peak_source": "derived: ALU pipe 148 SMs x 4 SMSPs x 16 lanes/clk (rt 2 clk/warp-instr, B300_MICROARCH.md) x max SM clock"},
        "e2e": None, "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
        "gpu_launches_per_step": launches_per_step,
    }
    return line, fam, conf, ok


def cpu_baseline_graph(fam, seconds, conf, ok):
    """The oracle's replay (plain C loops, one thread) on a bounded sample of
    the grid's vectors over the same validation set."""
    import numpy as np
    import oracle
    c = conf.cpu().numpy()
    o = ok.cpu().numpy()
    K, n = o.shape
    S = oracle.grid_size(K, GRAPH_Q)
    m = 4
    while True:
        idx = np.linspace(0, S - 1, m).astype(np.int64)
        bv = np.array([oracle.grid_vector(int(s), K, GRAPH_Q) for s in idx], np.int32)
        t = time.perf_counter()
        oracle.replay(c, o, GRAPH_Q, GRAPH_W, bvecs=bv)
        dt = time.perf_counter() - t
        if dt >= seconds / 3 or m >= S:
            break
        m = min(S, int(m * max(2.0, seconds / max(dt, 1e-3))))
    return {"value": m * n / dt, "unit": "replays/s", "cores": 1, "kind": "oracle",
            "sample": f"{m} of the {S} grid vectors (evenly spaced) x all {n} validation samples, "
                      f"fp64 C oracle (hso_replay), 1 thread, {dt:.1f} s"}


def synth_scaled(fam, **kw):
    from workload import synth
    return synth.scaled(fam, **kw)


def cpu_baseline_temperature(fam, seconds: float, val, labels):
    """The oracle's fit (fp64, bisection) on a bounded row sample of the same
    validation logits, repeated for ~`seconds`."""
    import numpy as np
    import oracle
    K = fam.K
    lab = labels.cpu().numpy()
    rows_all = [x.view(__import__("torch").int16).cpu().numpy().view(np.uint16) for x in val]
    m = 256
    t = time.perf_counter()
    for k in range(K):
        oracle.fit_temperature(rows_all[k][:m], lab[:m], n_classes=fam.C)
    dt = time.perf_counter() - t
    m = int(min(len(lab), max(m, m * seconds / max(dt, 1e-3))))
    t = time.perf_counter()
    for k in range(K):
        oracle.fit_temperature(rows_all[k][:m], lab[:m], n_classes=fam.C)
    dt = time.perf_counter() - t
    return {"value": K * m / dt, "unit": "rows/s", "cores": 1, "kind": "oracle",
            "sample": f"first {m} of {len(lab)} validation rows of each of the {K} stage models "
                      f"(same generator), fp64 C oracle (bisection on beta), 1 thread, {dt:.1f} s"}


# ---------------------------------------------------------------------------
# the oracle on the host cores (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------
def oracle_inputs(fam, frac_n: int, frac_val: int):
    """Host bytes of a bounded sample of the workload (same keyed generator)."""
    import numpy as np
    from workload import synth
    K = fam.K
    ids = np.arange(frac_n, dtype=np.int64)
    vids = np.arange(frac_val, dtype=np.int64) + synth.VAL_ID_BASE
    lab = synth.labels_np(fam.seed, vids, fam.L, fam.C).reshape(-1)
    vl = [synth.fam_logits_np(fam, k, vids, fam.dtype, L=fam.L, C=fam.C) for k in range(K)]
    rl = [synth.fam_logits_np(fam, k, ids, fam.dtype, L=fam.L, C=fam.C) for k in range(K)]
    return {"n": frac_n, "v": frac_val, "lab": lab, "vl": vl, "rl": rl}


def oracle_step(fam, inp):
    """One oracle step (the oracle as it stands, all host threads): validation
    confidences of every stage -> calibration -> cascade routing of the sample.
    Returns (seconds, requests routed)."""
    import numpy as np
    import oracle
    K, nv, n = fam.K, inp["v"], inp["n"]
    t = time.perf_counter()
    conf = np.empty((K - 1, nv))
    ok = np.empty((K, nv), np.uint8)
    for k in range(K):
        r = oracle.confidence(inp["vl"][k], nv, fam.L, fam.C, fam.C, fam.temps[k], kind=fam.kind,
                              reduce=fam.reduce, labels=inp["lab"], top_k=fam.top_k)
        ok[k] = r["correct"]
        if k < K - 1:
            conf[k] = r["conf"]
    cal = oracle.calibrate(conf, ok, fam.log2_bins)
    batch = np.arange(n, dtype=np.int64)
    for k in range(K):
        r = oracle.confidence(inp["rl"][k], len(batch), fam.L, fam.C, fam.C, fam.temps[k],
                              kind=fam.kind, reduce=fam.reduce, row_index=batch, top_k=fam.top_k)
        acc, dfr = oracle.route(r["conf"], float(np.float32(cal["t"][k])), k == K - 1)
        batch = batch[dfr]
    inp["last"] = {"vconf": conf, "vok": ok, "cal": cal}
    return time.perf_counter() - t, n


def cpu_parity(fam, inp, router):
    """Part of the cpu_baseline leg: the oracle's outputs of the timed sample
    against the GPU's outputs of the same requests (SURVEY 8(c) protocol).
      * validation confidences of the sample (1e-5 relative) and correct bits;
      * calibration (i): the oracle's D5 sweep on the GPU's confidences of the
        WHOLE validation shard must give the GPU's b bit-exactly; (ii) on its
        own confidences (when the sample is the whole shard): equal, or the
        samples that changed bin are counted;
      * routing: every sampled request's answering model under the GPU's
        thresholds equals the oracle cascade's, except near-threshold
        requests (|c - t_k| <= 1e-5 t_k at a stage they reach), counted per stage."""
    import numpy as np
    import oracle
    K, nv, n = fam.K, inp["v"], inp["n"]
    last = inp["last"]
    gv = router.vconf_all.view(K, fam.n_val).cpu().numpy().astype(np.float64)
    gok = router.vok.view(K, fam.n_val).cpu().numpy()
    oc = last["vconf"]
    err = np.abs(gv[: K - 1, :nv] - oc) / np.maximum(np.abs(oc), 1e-300)
    b_gpu = router.cal["b"].cpu().numpy()
    cal_i = oracle.calibrate(gv[: K - 1].astype(np.float32), gok, fam.log2_bins)
    out = {"validation_conf_max_rel_err": float(np.nanmax(err)) if err.size else 0.0,
           "validation_correct_bits_equal": bool(np.array_equal(gok[:, :nv], last["vok"])),
           "calibration_i_bit_exact": bool(np.array_equal(cal_i["b"], b_gpu))}
    if nv == fam.n_val:
        B = 1 << fam.log2_bins
        ob = np.where(np.isnan(oc), -1, np.minimum(B, np.floor(oc * B)))
        gb = np.where(np.isnan(gv[: K - 1]), -1, np.minimum(B, np.floor(gv[: K - 1] * B)))
        out["calibration_ii_equal"] = bool(np.array_equal(last["cal"]["b"], b_gpu))
        out["calibration_ii_samples_changed_bin"] = int((ob != gb).sum())
    # routing of the sampled requests (ids 0..n-1 of this shard)
    t = router.cal["t"].cpu().numpy().astype(np.float64)
    conf = np.stack([oracle.confidence(inp["rl"][k], n, fam.L, fam.C, fam.C, fam.temps[k], kind=fam.kind,
                                       reduce=fam.reduce, top_k=fam.top_k)["conf"] for k in range(K)])
    st_o = oracle.cascade(conf, t)
    st_g = np.full(n, -1, np.int64)
    counts = router.cascade.counts.cpu().numpy()
    for k in range(K):
        ids = router.cascade.outs[k]["acc_ids"][: int(counts[k][0])].cpu().numpy()
        ids = ids[ids < n]
        st_g[ids] = k
    near = np.zeros(n, bool)
    per = []
    for k in range(K - 1):
        nk = (st_o >= k) & (np.abs(conf[k] - t[k]) <= 1e-5 * t[k]) if np.isfinite(t[k]) else np.zeros(n, bool)
        per.append(int(nk.sum()))
        near |= nk
    out.update({"requests_checked": n, "near_threshold_per_stage": per,
                "routing_mismatches_excluding_near": int((st_o[~near] != st_g[~near]).sum()),
                "routing_mismatches_near": int((st_o[near] != st_g[near]).sum())})
    out["green"] = (out["validation_conf_max_rel_err"] <= 1e-5 and out["validation_correct_bits_equal"]
                    and out["calibration_i_bit_exact"] and out["routing_mismatches_excluding_near"] == 0)
    return out


def cpu_sample_sizes(fam, seconds: float):
    """Scale the oracle sample so one step takes ~`seconds` on this host (capped
    at the full per-GPU workload)."""
    n0 = min(fam.n, 1024)
    v0 = max(64, int(n0 * fam.n_val / fam.n))
    dt, _ = oracle_step(fam, oracle_inputs(fam, n0, v0))
    scale = max(1.0, seconds / max(dt, 1e-3))
    n = int(min(fam.n, n0 * scale))
    v = int(min(fam.n_val, max(64, n * fam.n_val / fam.n)))
    return n, v


def cpu_baseline(fam, seconds: float, router=None):
    """The oracle on the host cores, repeated over a bounded sample for ~`seconds`;
    with the GPU's router, the oracle's outputs of that sample are also checked
    against the GPU's (``parity``)."""
    n, v = cpu_sample_sizes(fam, seconds)
    inp = oracle_inputs(fam, n, v)
    tot, routed, reps = 0.0, 0, 0
    while tot < seconds and reps < 100:
        dt, r = oracle_step(fam, inp)
        tot += dt
        routed += r
        reps += 1
    out = {"value": routed / tot, "unit": "requests/s", "cores": os.cpu_count(), "kind": "oracle",
           "sample": f"{reps} x ({n} of {fam.n} requests + {v} of {fam.n_val} validation samples "
                     f"of {fam.name}, same generator), fp64 C oracle on {os.cpu_count()} threads, "
                     f"{tot:.1f} s"}
    if router is not None and fam.top_k == 0 and fam.L == 1:
        out["parity"] = cpu_parity(fam, inp, router)
    return out


def run_reference(args, world, rank):
    """--impl reference: the oracle as it stands, on host cores, K bounded steps."""
    if rank != 0:
        return None
    if args.config == "c2t":
        return run_reference_temperature(args, world)
    if args.config == "c2g":
        return run_reference_graph(args, world)
    fam = family(args.config)
    budget = 150.0 / max(1, args.steps + args.warmup)
    n, v = cpu_sample_sizes(fam, min(budget, 20.0))
    inp = oracle_inputs(fam, n, v)
    for _ in range(args.warmup):
        oracle_step(fam, inp)
    tot = 0.0
    routed = 0
    for _ in range(args.steps):
        dt, r = oracle_step(fam, inp)
        tot += dt
        routed += r
    value = routed / tot
    ms = tot / args.steps * 1e3
    sample = f"{n} of {fam.n} requests + {v} of {fam.n_val} validation samples of {fam.name} per step"
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "requests/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": fam.name, "description": CONFIG_TEXT[args.config],
                       "requests_per_gpu": fam.n, "validation_per_gpu": fam.n_val, "K": fam.K,
                       "classes": fam.C, "logits_dtype": fam.dtype,
                       "parallelism": "host cores (oracle)"},
            "cpu_baseline": {"value": value, "unit": "requests/s", "cores": os.cpu_count(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "requests/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def run_reference_temperature(args, world):
    """--impl reference --config c2t: the oracle's fit on a bounded row sample."""
    import numpy as np
    import oracle
    from workload import synth
    fam = family("c2")
    budget = min(10.0, 150.0 / max(1, args.steps + args.warmup))
    vids = np.arange(fam.n_val, dtype=np.int64) + synth.VAL_ID_BASE
    m = 128
    while True:
        lab = synth.labels_np(fam.seed, vids[:m], 1, fam.C).reshape(-1)
        rows = [synth.fam_logits_np(fam, k, vids[:m], "bf16", L=1, C=fam.C) for k in range(fam.K)]
        t = time.perf_counter()
        for k in range(fam.K):
            oracle.fit_temperature(rows[k], lab, n_classes=fam.C)
        dt = time.perf_counter() - t
        if dt >= budget / 4 or m >= fam.n_val:
            break
        m = min(fam.n_val, int(m * max(2.0, budget / max(dt, 1e-3))))
    for _ in range(args.warmup):
        for k in range(fam.K):
            oracle.fit_temperature(rows[k], lab, n_classes=fam.C)
    tot = 0.0
    for _ in range(args.steps):
        t = time.perf_counter()
        for k in range(fam.K):
            oracle.fit_temperature(rows[k], lab, n_classes=fam.C)
        tot += time.perf_counter() - t
    value = fam.K * m * args.steps / tot
    sample = f"first {m} of {fam.n_val} validation rows of each of the {fam.K} stage models per step"
    return {"impl": "reference", "metric": METRIC_TEMP, "value": value, "unit": "rows/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c2t_vit5_validation_temperature", "description": CONFIG_TEXT["c2t"],
                       "validation_per_gpu": fam.n_val, "K": fam.K, "classes": fam.C,
                       "logits_dtype": "bf16", "parallelism": "host core (oracle, 1 thread)"},
            "cpu_baseline": {"value": value, "unit": "rows/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_reference_graph(args, world):
    """--impl reference --config c2g: the oracle's replay of a bounded vector
    sample per step, on oracle confidences of the same validation set."""
    import numpy as np
    import oracle
    from workload import synth
    fam = family("c2")
    K, n = fam.K, fam.n_val
    vids = np.arange(n, dtype=np.int64) + synth.VAL_ID_BASE
    lab = synth.labels_np(fam.seed, vids, 1, fam.C).reshape(-1)
    conf = np.empty((K - 1, n))
    ok = np.empty((K, n), np.uint8)
    for k in range(K):
        bits = synth.fam_logits_np(fam, k, vids, "bf16", L=1, C=fam.C)
        r = oracle.confidence(bits, n, 1, fam.C, fam.C, fam.temps[k], labels=lab)
        ok[k] = r["correct"]
        if k < K - 1:
            conf[k] = r["conf"]
    S = oracle.grid_size(K, GRAPH_Q)
    budget = min(10.0, 150.0 / max(1, args.steps + args.warmup))
    m = 4
    while True:
        bv = np.array([oracle.grid_vector(int(s), K, GRAPH_Q)
                       for s in np.linspace(0, S - 1, m).astype(np.int64)], np.int32)
        t = time.perf_counter()
        oracle.replay(conf, ok, GRAPH_Q, GRAPH_W, bvecs=bv)
        dt = time.perf_counter() - t
        if dt >= budget / 3 or m >= S:
            break
        m = min(S, int(m * max(2.0, budget / max(dt, 1e-3))))
    for _ in range(args.warmup):
        oracle.replay(conf, ok, GRAPH_Q, GRAPH_W, bvecs=bv)
    tot = 0.0
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle.replay(conf, ok, GRAPH_Q, GRAPH_W, bvecs=bv)
        tot += time.perf_counter() - t
    value = m * n * args.steps / tot
    sample = f"{m} of the {S} grid vectors x all {n} validation samples per step"
    return {"impl": "reference", "metric": METRIC_GRAPH, "value": value, "unit": "replays/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c2g_vit5_grid_q4", "description": CONFIG_TEXT["c2g"],
                       "validation_per_gpu": n, "K": K, "log2_bins": GRAPH_Q,
                       "parallelism": "host core (oracle, 1 thread)"},
            "cpu_baseline": {"value": value, "unit": "replays/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "replays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _claim_stdout():
    """Route C-level stdout (NCCL's version banner, library prints) to stderr for
    the whole run; return a writer for the one JSON line on the real stdout."""
    sys.stdout.flush()
    real = os.dup(1)
    os.dup2(2, 1)

    def emit(line: str):
        os.write(real, (line + "\n").encode())

    return emit


def spawn_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: re-launch this script as N
    ranks (torch.distributed.run, one process per GPU, rendezvous on
    127.0.0.1); rank 0's JSON line is the output."""
    import socket
    import subprocess
    import torch
    if not (args.share_gpu or args.plumbing_check) and torch.cuda.device_count() < args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} needs {args.gpus} visible GPUs, "
                         f"found {torch.cuda.device_count()}")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def plumbing_check(world: int, rank: int):
    """--plumbing-check: the launcher and the host-side helpers of the
    multi-rank bench on CPU (gloo): what a peer group does once at set-up
    (all_gather_object of a 64-byte handle) and the max / sum over ranks the
    timing uses."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    handles = [None] * world
    mine = bytes([rank]) * 64
    if world > 1:
        dist.all_gather_object(handles, mine)
    else:
        handles = [mine]
    mx = max_over_ranks([float(rank), 10.0 - rank], world)
    sm = sum_over_ranks([float(rank + 1)], world)
    ok = all(h == bytes([r]) * 64 for r, h in enumerate(handles))
    if world > 1:
        barrier(world)
        dist.destroy_process_group()
    if rank != 0:
        return None
    return {"plumbing_check": True, "world": world, "handles_ok": ok, "max": mx, "sum": sm}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    emit = _claim_stdout()
    if world > 1 and args.gpus not in (1, world):
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE {world}: using {world}", file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    if args.plumbing_check:
        line = plumbing_check(world, rank)
        if line is not None:
            emit(json.dumps(line))
        return
    if args.impl == "reference":
        line = run_reference(args, world, rank)
        if line is not None:
            emit(json.dumps(line))
        return
    if (args.placement == "nccl" or args.force_dist) and world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ["WORLD_SIZE"] = "1"
        os.environ["RANK"] = "0"
        os.environ["LOCAL_RANK"] = "0"
    world, rank, local = init_dist(args, force=args.placement == "nccl" or args.force_dist)
    if args.config == "c2g":
        line, fam, conf, ok = run_graph(args, world, rank, local)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_graph(fam, args.cpu_seconds, conf, ok)
        if rank == 0:
            emit(json.dumps(line))
        return
    if args.config == "c2skip":
        line = run_skip(args, world, rank, local)
        if rank == 0:
            emit(json.dumps(line))
        return
    if args.config == "c2t":
        line, fam, val, labels = run_temperature(args, world, rank, local)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_temperature(fam, args.cpu_seconds, val, labels)
        if rank == 0:
            emit(json.dumps(line))
        return
    router = None
    if args.placement == "nccl":
        line, fam = run_nccl(args, world, rank, local)
    else:
        line, fam, *_, router = run_ours(args, world, rank, local)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(fam, args.cpu_seconds,
                                                router if args.layout == "dense" else None)
        emit(json.dumps(line))
    import torch.distributed as dist
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
