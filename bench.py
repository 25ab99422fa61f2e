#!/usr/bin/env python3
"""Benchmark of the B200 chunk step: reduce-scatter -> fused Adam -> all-gather
over the ZeRO-3 chunk shards of a planner layout (BASELINE.json metric
"chunk step GB/s (gather+RS+fused Adam) vs HBM/NVLink roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2|flat512 ...]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...     # CPU reference arm (oracle port)

One step = one pass of the data plane over every chunk of the workload with
inputs resident in HBM: per chunk RS (w>1), fused Adam on the owned shard
(with grad-norm/overflow statistics), AG (w>1). `value` = algorithmic bytes
of all ranks / max-over-ranks device time; `e2e` = the same
metric through the C-ABI with pinned HOST gradient / parameter buffers, the
H2D of the step's gradients and D2H of its parameters (and the grad-norm
readback) inside the timed region.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")
PEAKS_FILE = os.path.join(REPO, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0      # B200_PROFILING.md fallback
NVLINK_GBS = 770.0             # measured peer copy per direction (B200_PROFILING.md)

WORKLOADS = {
    # name: (description, layout source)
    "cfg2": ("GPT-2 1.5B (h1600 L48 25 heads) b8, 3x1GiB chunks, all persistent, ZeRO-3 sharded",
             "layout:gpt2-1.5b_b8"),
    "cfg1": ("gpt2-1b b2 (reference test model), 4x512MiB chunks, all persistent",
             "layout:gpt2-1b_b2"),
    "cfg3": ("gpt2-10b b8, 49x512MiB chunks, all persistent on one GPU (158 GB of chunk state)",
             "layout:gpt2-10b_b8"),
    "flat32": ("flat 32 MiB chunk sweep point", "flat:33554432"),
    "flat64": ("flat 64 MiB chunk", "flat:67108864"),
    "flat128": ("flat 128 MiB chunk", "flat:134217728"),
    "flat256": ("flat 256 MiB chunk", "flat:268435456"),
    "flat512": ("flat 512 MiB chunk", "flat:536870912"),
    "cfg2flat": ("cfg2's 1,557,608,000 parameters as ONE flat chunk (per-launch overhead "
                 "diagnostic)", "flat:3115216000"),
}


def chunk_numels(workload: str) -> tuple[list[int], str]:
    desc, src = WORKLOADS[workload]
    kind, arg = src.split(":", 1)
    if kind == "flat":
        return [int(arg) // 2], desc
    # The chunk table comes from the planner (pack_chunks / chunk_size_search),
    # run here; its output is byte-identical to the reference's
    # (tests/test_planner.py against tests/golden/).
    from paper_2406_08334_b200 import planner
    layout = planner.layout_for(arg)
    return [c["used_bytes"] // layout["bytes_per_param"] for c in layout["chunks"]], desc


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every 20 ms DURING
    the timed region (the profiling recipe's nvidia-smi clocks line, read via
    nvidia-ml-py so no subprocess output buffering can lose samples)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index, self.samples, self.stop = index, [], threading.Event()
        self.max_mhz, self.error = None, None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.index]) if vis else self.index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.nvml = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as e:  # noqa: BLE001
            self.error = repr(e)
        return self

    def _run(self):
        while not self.stop.is_set():
            try:
                sm = self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM)
                rs = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception as e:  # noqa: BLE001
                self.error = repr(e)
                return
            time.sleep(0.02)

    def __exit__(self, *exc):
        self.stop.set()
        if hasattr(self, "thread"):
            self.thread.join(timeout=2)

    def summary(self):
        sm = [s for s, _ in self.samples]
        reasons = set()
        for _, rs in self.samples:
            for bit, name in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
               "reasons": sorted(reasons), "samples": len(sm)}
        if self.error:
            out["error"] = self.error
        return out


def dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def make_comm(world, rank):
    """NCCL communicator of libptk; the unique id travels over the gloo group."""
    from paper_2406_08334_b200 import _native as nat
    import torch
    import torch.distributed as dist
    if world == 1:
        return None
    uid = (ctypes.c_uint8 * nat.PTK_UNIQUE_ID_BYTES)()
    if rank == 0:
        nat.lib.ptk_comm_unique_id(uid)
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
    dist.broadcast(t, 0)
    uid = (ctypes.c_uint8 * nat.PTK_UNIQUE_ID_BYTES)(*t.tolist())
    comm = ctypes.c_void_p()
    nat.lib.ptk_comm_init(ctypes.byref(comm), world, rank, uid)
    return comm


def traffic_from_profiles(workload):
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# ------------------------------------------------------------------ GPU arm --

def run_gpu(args):
    import torch
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet, stream_handle, vp

    world, rank, local = dist_setup()
    mode = args.exchange
    if mode == "auto":
        mode = "fused" if world > 1 else "nccl"
    if args.shared_device:
        # flow validation on a one-GPU box: every rank on cuda:0, peers mapped
        # through cudaIpc as on an NVLink node; NCCL refuses duplicate devices,
        # so only the fused exchange runs and the timings are not a bench value
        if mode != "fused":
            raise SystemExit("--shared-device needs --exchange fused")
        local = 0
        args.train_steps = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numels, desc = chunk_numels(args.workload)
    comm = None if args.shared_device else make_comm(world, rank)
    cs = ChunkSet(numels, world=world, rank=rank, device=dev, mode=mode, comm=comm)
    stream = torch.cuda.current_stream()
    cs.init_synthetic()
    cs.fill_grads(0)
    if mode == "fused":
        if world > 1:
            cs.attach_ipc_peers()
        else:
            cs.attach_virtual_peers([cs])
    hyper = AdamHyper(lr=1e-3, weight_decay=0.0)
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        cs.step(hyper)
    torch.cuda.synchronize()
    barrier(world)

    # The K timed steps. With --graph (default at N=1) they are captured once
    # into a CUDA graph (each step with its own step number, so replaying it
    # once performs exactly steps n+1..n+K) and the timed region is one replay:
    # small chunks are then bound by the device, not by host launch latency.
    use_graph = args.graph and world == 1
    launches0 = nat.launch_count()
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(args.steps):
                cs.step(hyper)
        torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier(world)
        start.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for _ in range(args.steps):
                cs.step(hyper)
        end.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = nat.launch_count() - launches0
    del graph
    ms = start.elapsed_time(end) / args.steps
    ms_max = max_over_ranks(ms, world)
    bytes_rank = cs.algorithmic_hbm_bytes()
    total_bytes = bytes_rank * world  # every rank moves the same algorithmic bytes
    value = total_bytes / (ms_max * 1e-3) / 1e9

    # Dominant kernel, timed per launch with events on its own stream.
    kern = time_dominant_kernel(cs, hyper, stream, world, reps=max(1, min(args.steps, 5)),
                                use_graph=use_graph)
    hbm_peak, peak_kind = load_peaks()

    e2e = run_e2e(cs, hyper, args, world) if not args.no_e2e else None
    sumsq, nonfinite = cs.grad_stats()
    nvl_bytes_rank = cs.algorithmic_nvlink_bytes()
    if mode == "fused" and world > 1:
        torch.cuda.synchronize()
        barrier(world)   # no rank unmaps / frees while a peer may still store into it
        cs.close_ipc_peers()
    del cs
    torch.cuda.empty_cache()
    train = train_offload = None
    if args.train_steps > 0 and args.workload in TRAIN_MODELS:
        train = run_train(args, world, rank, dev, comm)
        if args.offload_persist >= 0:
            train_offload = run_train(args, world, rank, dev, comm,
                                      n_persist=args.offload_persist,
                                      n_buffer=args.offload_buffers)
    copy_peak = live_copy_peak()

    result = None
    if rank == 0:
        cpu = None if args.no_cpu_baseline or world > 1 else cpu_baseline(numels, args)
        result = {
            "metric": "chunk step GB/s (gather+RS+fused Adam) vs HBM/NVLink roofline",
            "value": round(value, 2),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_max, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32 (Adam state) / bf16 (grads, params)",
            "data": "synthetic (counter-based uniform; SURVEY §8(d) seeds)",
            "config": {
                "workload": f"{args.workload}: {desc}",
                "params": sum(numels),
                "chunks": len(numels),
                "chunk_params": numels,
                "exchange": ({"nccl": "nccl RS/AG (in place)",
                              "fused": "fused RS->Adam->AG kernel over NVLink peer memory"}[mode]
                             if world > 1 else f"none (w=1, {mode} path)"),
                "parallelism": f"zero3-dp{world}",
                "timed_steps": ("one CUDA-graph replay holding the K steps" if use_graph
                                else "K host-launched steps"),
                "l2": "inputs larger than L2 (%.1f GB touched per step)" % (bytes_rank / 1e9),
                "algorithmic_bytes_per_step_per_rank": bytes_rank,
                "nvlink_bytes_per_step_per_rank": nvl_bytes_rank,
                **({"shared_device_validation": "all ranks on cuda:0: flow check, not a bench value"}
                   if args.shared_device else {}),
            },
            "roofline": dict(roofline(kern, hbm_peak, peak_kind, args.workload),
                             live_copy_gbs_this_box=copy_peak,
                             frac_of_live_copy=round(kern["hbm_bytes"] / (kern["ms"] * 1e-3) /
                                                     1e9 / copy_peak, 4)),
            "e2e": e2e,
            "train": train,
            "train_offload": train_offload,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "grad_stats": {"sumsq": sumsq, "nonfinite": nonfinite},
            "cpu_baseline": cpu,
        }
    if comm is not None:
        nat.lib.ptk_comm_destroy(comm)
    return result


def time_dominant_kernel(cs, hyper, stream, world, reps, use_graph=False):
    """Average launch duration of the step's dominant kernel (CUDA events on
    the stream it is launched on) and its algorithmic bytes per launch.
    Eager: events around every launch (includes its launch latency). Graph:
    `reps` passes over the chunks captured back to back, events around one
    replay on the launching stream, divided by the number of launches."""
    import torch
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import stream_handle, vp
    cfg = hyper.config(cs.step_count + 1, world)
    ms, hbm, nvl = 0.0, 0, 0
    torch.cuda.synchronize()
    if use_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            sh = stream_handle(None)
            for _ in range(reps):
                for c in cs.chunks:
                    _launch_dominant(cs, c, cfg, world, sh)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        del g
    else:
        sh = stream_handle(stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in cs.chunks]
        for _ in range(reps):
            for c, (e0, e1) in zip(cs.chunks, ev):
                e0.record(stream)
                _launch_dominant(cs, c, cfg, world, sh)
                e1.record(stream)
            torch.cuda.synchronize()
            ms += sum(e0.elapsed_time(e1) for e0, e1 in ev)
    for c in cs.chunks:
        p, w = c.numel, world
        if cs.mode == "fused":
            # local state 28P/w + grad shard reads 2P/w from each of w ranks
            # + param shard writes to w ranks (counted once per byte moved)
            hbm += 28 * p // w + 2 * p * (w - 1) // w * 2
            nvl += 2 * p * (w - 1) // w
        else:
            hbm += 28 * p // w
    hbm, nvl = hbm * reps, nvl * reps
    n = reps * len(cs.chunks)
    name = (nat.raw.ptk_fused_kernel_name().decode() if cs.mode == "fused"
            else "chunk_adam_tma_kernel (" + nat.raw.ptk_adam_kernel_name().decode() + ")")
    return {"kernel": name, "ms": ms, "hbm_bytes": hbm, "nvl_bytes": nvl, "launches": n,
            "world": world, "timing": "graph of back-to-back launches" if use_graph
            else "events around each launch"}


def _launch_dominant(cs, c, cfg, world, sh):
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import vp
    i = c.chunk_id
    if cs.mode == "fused":
        nat.lib.ptk_fused_rs_adam_ag(ctypes.byref(cfg), cs.peer_grad_ptrs[i],
                                     cs.peer_param_ptrs[i], world, cs.rank, c.shard,
                                     vp(c.master), vp(c.exp_avg), vp(c.exp_avg_sq),
                                     vp(cs.stats), vp(cs.workspace), sh)
    else:
        nat.lib.ptk_chunk_adam(ctypes.byref(cfg), vp(c.master), vp(c.exp_avg),
                               vp(c.exp_avg_sq), vp(c.grad_shard()), vp(c.param_shard()),
                               c.shard, vp(cs.stats), vp(cs.workspace), None, None, sh)


def roofline(k, hbm_peak, peak_kind, workload):
    t_hbm = k["hbm_bytes"] / (hbm_peak * 1e9)
    t_nvl = k["nvl_bytes"] / (NVLINK_GBS * 1e9)
    nvl_bound = t_nvl > t_hbm
    sec = k["ms"] * 1e-3
    achieved = (k["nvl_bytes"] if nvl_bound else k["hbm_bytes"]) / sec / 1e9
    peak = NVLINK_GBS if nvl_bound else hbm_peak
    return {"bound": "nvlink" if nvl_bound else "hbm", "kernel": k["kernel"],
            "achieved": round(achieved, 1), "peak": peak,
            "peak_kind": "measured peer copy per direction (B200_PROFILING.md)" if nvl_bound
            else peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": traffic_from_profiles(workload),
            "bytes_per_launch": (k["nvl_bytes"] if nvl_bound else k["hbm_bytes"]) // k["launches"],
            "ms_per_launch": round(k["ms"] / k["launches"], 4),
            "launch_timing": k["timing"],
            "frac_of_8tbs_spec": None if nvl_bound else round(achieved / 8000.0, 4)}


def live_copy_peak():
    """This box's HBM copy bandwidth, measured like MEASURED_PEAKS.json
    ('b.copy_(a) over 1 Gi bf16 elements, read+write bytes, best of 10'), to
    separate box-to-box HBM variance from kernel quality."""
    import torch
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return round(2 * 2 * (1 << 30) / (best * 1e-3) / 1e9, 1)


TRAIN_MODELS = {"cfg2": "gpt2-1.5b_b8", "cfg1": "gpt2-1b_b2"}


def run_train(args, world, rank, dev, comm, n_persist=None, n_buffer=0):
    """tokens/s of a full training iteration of the workload's model (cfg2:
    GPT-2 1.5B b8; cfg1: the reference's test model gpt2-1b b2; seq 1024)
    whose parameters live in the planner's chunk buffers:
    forward + backward in PyTorch (bf16 GEMMs / SDPA), then the chunk step
    (RS -> fused Adam -> AG) through the C-ABI. With n_persist < n_chunk the
    remaining chunks are non-persistent: pinned host shards fetched into
    n_buffer device slots, drained to the host Adam during backward (the
    iteration's time includes the last host update). Random-init weights,
    synthetic tokens; CUDA-event time over the timed iterations, max over ranks."""
    import torch
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step
    name = TRAIN_MODELS[args.workload]
    trace = planner.trace_for(name)
    layout = planner.layout_for(name)
    numels = [c["used_bytes"] // layout["bytes_per_param"] for c in layout["chunks"]]
    np_ = len(numels) if n_persist is None else n_persist
    cs = ChunkSet(numels[:np_], world=world, rank=rank, device=dev, mode="nccl", comm=comm)
    pool = (ChunkPool(numels, np_, n_buffer, world=world, rank=rank, comm=comm, device=dev)
            if np_ < len(numels) else None)
    shape = GPT2Shape.from_trace(trace)
    model = ChunkedGPT2(shape, layout, cs, trace["ops"], pool=pool)
    model.init_weights(seed=0)
    batch = int(trace["meta"]["batch_size"])
    n_iter = args.warmup + args.train_steps
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    # learnable synthetic stream (next token = token + 1) so the loss is a sanity signal
    tokens = torch.randint(0, shape.vocab, (n_iter, batch, shape.seq), device=dev, generator=gen)
    targets = (tokens + 1) % shape.vocab
    hyper = AdamHyper(lr=1e-4, weight_decay=0.01, adamw=True)
    stream = torch.cuda.current_stream()
    losses = []
    overlap = args.train_overlap
    graphed = None
    if args.train_graph and pool is None:
        from paper_2406_08334_b200.train import GraphedTrainStep
        graphed = GraphedTrainStep(model, tokens[0], targets[0])

    def one(i):
        if graphed is not None:
            return graphed(tokens[i], targets[i], hyper)
        return train_step(model, tokens[i], targets[i], hyper, overlap=overlap)

    for i in range(args.warmup):
        losses.append(one(i))
    torch.cuda.synchronize()
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.warmup, n_iter):
        losses.append(one(i))
    if pool is not None:
        pool.finish_step()  # the last host updates belong to the timed iterations
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(t0.elapsed_time(t1) / args.train_steps, world)
    loss_vals = [float(x) for x in losses]
    out = {"tokens_per_s": round(batch * shape.seq * world / (ms * 1e-3), 1),
           "ms_per_iter": round(ms, 3), "iters": args.train_steps,
           "model": f"{name}: GPT-2 h{shape.hidden} L{shape.blocks} {shape.heads} heads, "
                    f"{sum(numels) / 1e9:.2f} B params (tied, parameter-free final LN: the trace has "
                    f"no ln_f), b{batch} s{shape.seq} per rank, bf16 compute, fp32 master/m/v in chunks",
           "plan": {"n_chunk": len(numels), "n_persist": np_, "n_buffer": n_buffer if pool else 0},
           "loss_first": round(loss_vals[0], 4), "loss_last": round(loss_vals[-1], 4),
           "chunk_step": ("per chunk on a side stream as its gradients complete (overlapping "
                          "the backward)" if overlap else "after the backward"),
           "forward_backward": ("one CUDA-graph replay (GraphedTrainStep)" if graphed is not None
                                else "host-launched"),
           "data": "synthetic tokens (uniform ids, target = id + 1), random init"}
    if pool is not None:
        out["offload"] = {"pinned_host_GB": round(pool.host_bytes / 1e9, 3),
                          "buffer_GB": round(pool.device_bytes / 1e9, 3),
                          "fetches": pool.counters["fetch"], "evictions": pool.counters["evict"],
                          "h2d_GB": round(pool.counters["h2d_bytes"] / 1e9, 2),
                          "d2h_GB": round(pool.counters["d2h_bytes"] / 1e9, 2)}
    del model, cs, pool
    torch.cuda.empty_cache()
    return out


def run_e2e(cs, hyper, args, world):
    """Same step through the C-ABI with HOST buffers: per chunk piece, pinned
    H2D of the gradients (h2d stream) -> fused Adam (compute stream) -> pinned
    D2H of the updated bf16 parameters (d2h stream); events chain the three
    streams so the copies of piece i+1 / i-1 overlap the update of piece i."""
    import torch
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import stream_handle, vp

    piece = args.e2e_piece
    comp = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    # w = 1: the rank's shard is the chunk. w > 1: each rank hands in its
    # full local gradient chunk and gets the full gathered parameter chunk
    # back (what a ZeRO-3 caller's backward produces / forward consumes).
    span = (lambda c: c.shard) if world == 1 else (lambda c: c.n_pad)
    host_g = [torch.empty(span(c), dtype=torch.bfloat16, pin_memory=True) for c in cs.chunks]
    host_p = [torch.empty(span(c), dtype=torch.bfloat16, pin_memory=True) for c in cs.chunks]
    host_stats = torch.empty(2, dtype=torch.float64, pin_memory=True)
    for hg, c in zip(host_g, cs.chunks):
        hg.copy_((c.grad_shard() if world == 1 else c.grad).cpu())
    sc, sh, sd = stream_handle(comp), stream_handle(h2d), stream_handle(d2h)

    def one_step_fused():
        # all local gradient chunks in, then the fused RS->Adam->AG step
        # (peer barriers inside), then the gathered parameters out
        h2d.wait_stream(comp)
        for c, hg in zip(cs.chunks, host_g):
            nat.lib.ptk_memcpy_h2d_async(vp(c.grad), ctypes.c_void_p(hg.data_ptr()), 2 * c.n_pad, sh)
        comp.wait_stream(h2d)
        cs.step(hyper, stream=comp)
        d2h.wait_stream(comp)
        for c, hp in zip(cs.chunks, host_p):
            nat.lib.ptk_memcpy_d2h_async(ctypes.c_void_p(hp.data_ptr()), vp(c.param), 2 * c.n_pad, sd)
        comp.wait_stream(d2h)
        nat.lib.ptk_memcpy_d2h_async(vp(host_stats), vp(cs.stats), 16, sc)

    def one_step_sharded():
        if cs.mode == "fused":
            return one_step_fused()
        cs.step_count += 1
        cfg = hyper.config(cs.step_count, world)
        nat.lib.ptk_stats_reset(vp(cs.stats), sc)
        h2d.wait_stream(comp)
        for c, hg, hp in zip(cs.chunks, host_g, host_p):
            e_in, e_up = torch.cuda.Event(), torch.cuda.Event()
            nat.lib.ptk_memcpy_h2d_async(vp(c.grad), ctypes.c_void_p(hg.data_ptr()), 2 * c.n_pad, sh)
            e_in.record(h2d)
            comp.wait_event(e_in)
            nat.lib.ptk_chunk_reduce_scatter(cs.comm, vp(c.grad), c.shard, 0, sc)
            nat.lib.ptk_chunk_adam(ctypes.byref(cfg), vp(c.master), vp(c.exp_avg),
                                   vp(c.exp_avg_sq), vp(c.grad_shard()), vp(c.param_shard()),
                                   c.shard, vp(cs.stats), vp(cs.workspace), None, None, sc)
            nat.lib.ptk_chunk_allgather(cs.comm, vp(c.param), c.shard, 0, sc)
            e_up.record(comp)
            d2h.wait_event(e_up)
            nat.lib.ptk_memcpy_d2h_async(ctypes.c_void_p(hp.data_ptr()), vp(c.param), 2 * c.n_pad, sd)
        comp.wait_stream(d2h)
        nat.lib.ptk_memcpy_d2h_async(vp(host_stats), vp(cs.stats), 16, sc)

    def one_step():
        if world > 1:
            return one_step_sharded()
        cs.step_count += 1
        cfg = hyper.config(cs.step_count, world)
        nat.lib.ptk_stats_reset(vp(cs.stats), sc)
        for c, hg, hp in zip(cs.chunks, host_g, host_p):
            # at least ~8 pieces per chunk so copies overlap the update even
            # for small chunks (multiple of 12288 elements: whole TMA tiles)
            pc = min(piece, max(1 << 20, -(-c.shard // 8 // 12288) * 12288))
            for lo in range(0, c.shard, pc):
                n = min(pc, c.shard - lo)
                g_dev = c.grad_shard()[lo:lo + n]
                p_dev = c.param_shard()[lo:lo + n]
                e_in, e_up = torch.cuda.Event(), torch.cuda.Event()
                h2d.wait_stream(comp) if lo == 0 and c.chunk_id == 0 else None
                nat.lib.ptk_memcpy_h2d_async(vp(g_dev), ctypes.c_void_p(hg.data_ptr() + 2 * lo),
                                             2 * n, sh)
                e_in.record(h2d)
                comp.wait_event(e_in)
                nat.lib.ptk_chunk_adam(ctypes.byref(cfg), vp(c.master[lo:lo + n]),
                                       vp(c.exp_avg[lo:lo + n]), vp(c.exp_avg_sq[lo:lo + n]),
                                       vp(g_dev), vp(p_dev), n, vp(cs.stats), vp(cs.workspace),
                                       None, None, sc)
                e_up.record(comp)
                d2h.wait_event(e_up)
                nat.lib.ptk_memcpy_d2h_async(ctypes.c_void_p(hp.data_ptr() + 2 * lo), vp(p_dev),
                                             2 * n, sd)
        comp.wait_stream(d2h)
        nat.lib.ptk_memcpy_d2h_async(vp(host_stats), vp(cs.stats), 16, sc)

    link = pcie_ceiling(h2d, d2h, comp)
    steps = max(1, min(args.steps, args.e2e_steps))
    for _ in range(max(1, args.warmup)):
        one_step()
    torch.cuda.synchronize()
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(comp)
    for _ in range(steps):
        one_step()
    t1.record(comp)
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(t0.elapsed_time(t1) / steps, world)
    h2d_bytes = sum(2 * span(c) for c in cs.chunks)
    d2h_bytes = sum(2 * span(c) for c in cs.chunks) + 16
    value = cs.algorithmic_hbm_bytes() * world / (ms * 1e-3) / 1e9
    return {"value": round(value, 2), "unit": "GB/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
            "steps": steps,
            # the bound of this number is the host link, not HBM: the same
            # bytes moved by bare concurrent pinned copies (no kernel)
            "pcie_ceiling": {**link, "copy_only_ms": round(
                max(h2d_bytes / link["h2d_gbs_concurrent"], d2h_bytes / link["d2h_gbs_concurrent"])
                / 1e6, 3)},
            "frac_of_pcie_ceiling": round(
                max(h2d_bytes / link["h2d_gbs_concurrent"],
                    d2h_bytes / link["d2h_gbs_concurrent"]) / 1e6 / ms, 3),
            "path": ("C-ABI ptk_memcpy_h2d_async -> ptk_chunk_adam -> ptk_memcpy_d2h_async, "
                     f"pinned host buffers, pieces of min({piece}, max(1 Mi, chunk/8)) elements "
                     "on 3 streams") if world == 1 else
                    ("C-ABI: H2D local grad chunks -> ptk_peer_barrier -> ptk_fused_rs_adam_ag "
                     "-> ptk_peer_barrier -> D2H gathered params") if cs.mode == "fused" else
                    ("C-ABI per chunk: H2D local grad chunk -> ptk_chunk_reduce_scatter -> "
                     "ptk_chunk_adam -> ptk_chunk_allgather -> D2H gathered params, 3 streams")}


def pcie_ceiling(h2d, d2h, comp, nbytes=1 << 30, reps=3):
    """Concurrent pinned H2D + D2H of nbytes each (both directions at once,
    as in the e2e step): the host-link ceiling the e2e number is bound by."""
    import torch
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import stream_handle
    hsrc = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    hdst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    da = torch.empty(nbytes, dtype=torch.uint8, device=torch.cuda.current_device())
    db = torch.empty_like(da)
    best = None
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        h2d.wait_stream(comp)
        d2h.wait_stream(comp)
        ev[0].record(h2d)
        ev[2].record(d2h)
        nat.lib.ptk_memcpy_h2d_async(ctypes.c_void_p(da.data_ptr()), ctypes.c_void_p(hsrc.data_ptr()),
                                     nbytes, stream_handle(h2d))
        nat.lib.ptk_memcpy_d2h_async(ctypes.c_void_p(hdst.data_ptr()), ctypes.c_void_p(db.data_ptr()),
                                     nbytes, stream_handle(d2h))
        ev[1].record(h2d)
        ev[3].record(d2h)
        torch.cuda.synchronize()
        up, down = ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])
        cur = (nbytes / up / 1e6, nbytes / down / 1e6)
        best = cur if best is None or sum(cur) > sum(best) else best
    del hsrc, hdst, da, db
    return {"h2d_gbs_concurrent": round(best[0], 2), "d2h_gbs_concurrent": round(best[1], 2),
            "bytes_each_way": nbytes}


# ------------------------------------------------------------------ CPU arm --

def cpu_sample_step(n: int, threads: int):
    """One bounded sample of the chunk step on the host: oracle fp32 Adam over
    n parameters (28 B/param algorithmic bytes, w = 1)."""
    import numpy as np
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle_lib as ol
    master = ol.fill_f32(n, 0, 0.05)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    g = ol.fill_bf16(n, 1, 1e-3)
    out = np.empty(n, np.uint16)
    return ol, master, m, v, g, out


def cpu_baseline(numels, args):
    import numpy as np
    n = min(args.cpu_sample, sum(numels))
    ol, master, m, v, g, out = cpu_sample_step(n, 0)
    times = []
    for step in range(1, 4):
        s = ol.scalars(step=step)
        t0 = time.perf_counter()
        ol.adam_step(s, master, m, v, g, out)
        times.append(time.perf_counter() - t0)
    best = min(times)
    return {"value": round(28 * n / best / 1e9, 3), "unit": "GB/s", "cores": ol.num_threads(),
            "kind": "port",
            "sample": f"oracle fp32 Adam step over {n} params of the workload (28 B/param), "
                      "best of 3, OpenMP over all host threads"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    numels, desc = chunk_numels(args.workload)
    n = min(args.cpu_sample, sum(numels))
    ol, master, m, v, g, out = cpu_sample_step(n, 0)
    for step in range(1, args.warmup + 1):
        ol.adam_step(ol.scalars(step=step), master, m, v, g, out)
    t0 = time.perf_counter()
    for step in range(args.warmup + 1, args.warmup + args.steps + 1):
        ol.adam_step(ol.scalars(step=step), master, m, v, g, out)
    dt = (time.perf_counter() - t0) / args.steps
    value = 28 * n / dt / 1e9
    sample = (f"oracle port (oracle/chunk_step.c) fp32 Adam over a {n}-param sample of the "
              f"workload per step, w=1 data plane (the reference memplan never executes the "
              f"data plane, SPEC.md:514), OpenMP over all host threads")
    return {"impl": "reference", "metric":
            "chunk step GB/s (gather+RS+fused Adam) vs HBM/NVLink roofline",
            "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (Adam state) / bf16",
            "data": "synthetic", "config": {"workload": f"{args.workload}: {desc}",
                                            "sample_params": n},
            "cpu_baseline": {"value": round(value, 3), "unit": "GB/s",
                             "cores": ol.num_threads(), "kind": "port", "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ptk", choices=["ptk", "reference"])
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl", "fused"],
                    help="N>1 chunk exchange: the single fused RS->Adam->AG kernel over NVLink "
                         "peer memory (auto at N>1), or NCCL RS/AG + chunk Adam (the library "
                         "baseline; auto at N=1, where there is no exchange)")
    ap.add_argument("--cpu-sample", type=int, default=64 * 1024 * 1024)
    ap.add_argument("--e2e-piece", type=int, default=32 * 1024 * 1024)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--offload-persist", type=int, default=1,
                    help="also time training with chunks >= this index non-persistent "
                         "(pinned host + host Adam); -1 = skip")
    ap.add_argument("--offload-buffers", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--train-steps", type=int, default=10,
                    help="timed iterations of the end-to-end cfg2 training step (tokens/s); 0 = skip")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--train-graph", action=argparse.BooleanOptionalAction, default=True,
                    help="training (all chunks persistent): forward + backward as one CUDA-graph "
                         "replay, chunk step eager (default; --no-train-graph: host-launched)")
    ap.add_argument("--train-overlap", action=argparse.BooleanOptionalAction, default=False,
                    help="training: issue each persistent chunk's step on a side stream as soon "
                         "as its gradients are complete")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=True,
                    help="N=1: time the K steps as one replay of a CUDA graph holding them "
                         "(default); --no-graph: host-launched steps")
    ap.add_argument("--shared-device", action="store_true",
                    help="validation only: all ranks on cuda:0 (one-GPU box), fused exchange "
                         "over cudaIpc; exercises the N>1 flow, its timings are not a bench value")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        res = run_reference(args)
    else:
        res = run_gpu(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
