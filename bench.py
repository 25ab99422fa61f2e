#!/usr/bin/env python3
"""Benchmark of the B200 chunk step: reduce-scatter -> fused Adam -> all-gather
over the ZeRO-3 chunk shards of a planner layout (BASELINE.json metric
"chunk step GB/s (gather+RS+fused Adam) vs HBM/NVLink roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2|flat512 ...]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...     # CPU reference arm (oracle port)

`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks (127.0.0.1); under torchrun WORLD_SIZE must equal N.

One step = one pass of the data plane over every chunk of the workload with
inputs resident in HBM. At N = 1: one launch of the chunk-table Adam over all
chunks (with grad-norm / overflow statistics). At N > 1 BOTH exchanges are
measured and reported: the fused RS -> Adam -> AG kernel over NVLink peer
memory (one launch per step between two peer barriers) and the library
baseline (NCCL reduce-scatter per chunk, chunk-table Adam on the owned
shards, NCCL all-gather per chunk); `value` is the faster of the legs that
completed (`exchange` names it). `value` = BASELINE.md §3 algorithmic HBM
bytes of all ranks / max-over-ranks device time (the same accounting for
every exchange and for the CPU arm); the roofline uses each kernel's own
bytes. `e2e` = the same metric through the C-ABI with pinned HOST gradient /
parameter buffers, H2D of the step's gradients and D2H of its parameters
(and the statistics) inside the timed region.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time
import traceback

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")
PEAKS_FILE = os.path.join(REPO, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0      # B200_PROFILING.md fallback
NVLINK_GBS = 770.0             # measured peer copy per direction (B200_PROFILING.md)
METRIC = "chunk step GB/s (gather+RS+fused Adam) vs HBM/NVLink roofline"
CFG2_PARAMS = 1_557_608_000    # GPT-2 1.5B (SURVEY §8(a) golden layout)

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
# cfg5 as a model: cfg2's parameters packed into flat chunks of S MiB (the
# chunk-size sweep of one model: 93 chunks at 32 MiB ... 6 at 512 MiB)
for _mib in (32, 64, 128, 256, 512):
    WORKLOADS[f"cfg2x{_mib}"] = (f"cfg2's 1,557,608,000 parameters in flat {_mib} MiB chunks "
                                 "(chunk-size sweep of one model)", f"split:{_mib << 20}")


def chunk_numels(workload: str) -> tuple[list[int], str]:
    desc, src = WORKLOADS[workload]
    kind, arg = src.split(":", 1)
    if kind == "flat":
        return [int(arg) // 2], desc
    if kind == "split":
        per = int(arg) // 2
        full, rem = divmod(CFG2_PARAMS, per)
        return [per] * full + ([rem] if rem else []), desc
    # The chunk table comes from the planner (pack_chunks / chunk_size_search),
    # run here; its output is byte-identical to the reference's
    # (tests/test_planner.py against tests/golden/).
    from paper_2406_08334_b200 import planner
    layout = planner.layout_for(arg)
    return [c["used_bytes"] // layout["bytes_per_param"] for c in layout["chunks"]], desc


# ------------------------------------------------------ algorithmic bytes --

def metric_hbm_bytes(numels, w: int) -> int:
    """Per-rank HBM bytes of one chunk step, BASELINE.md §3 / SURVEY §8(d):
    28P/w (Adam) + 2P(w-1)/w (AG receive) + 2P + 2P/w (RS read / write);
    w = 1 -> 28P. The accounting of `value` for every exchange and arm."""
    tot = 0
    for p in numels:
        tot += 28 * p // w
        if w > 1:
            tot += 2 * p * (w - 1) // w + 2 * p + 2 * p // w
    return tot


def required_hbm_bytes(numels, w: int, mode: str) -> int:
    """Per-rank HBM bytes the exchange actually has to move. fused: the owned
    shard's state and own grad/param (28P/w) plus the peers' reads of this
    rank's gradients and writes of their parameter shards (4P(w-1)/w);
    nccl: the chunk-table Adam on the owned shards (28P/w) -- the NCCL
    kernels' own traffic is the rest of metric_hbm_bytes."""
    if mode == "fused":
        return sum(28 * p // w + 4 * p * (w - 1) // w for p in numels)
    return sum(28 * p // w for p in numels)


def nvlink_bytes(numels, w: int) -> int:
    """Per-rank NVLink bytes per direction: 4P(w-1)/w (RS + AG, bf16)."""
    return sum(4 * p * (w - 1) // w for p in numels)


def dominant_kernel_bytes(numels, w: int, mode: str) -> tuple[int, int]:
    """(HBM, NVLink-per-direction) bytes of ONE launch of the step's
    dominant kernel: the fused table kernel (fused) or the chunk-table Adam
    over the owned shards (nccl / w = 1)."""
    if mode == "fused":
        return required_hbm_bytes(numels, w, "fused"), nvlink_bytes(numels, w)
    return required_hbm_bytes(numels, w, "nccl"), 0


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


# ------------------------------------------------------------ process group --

def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """`--gpus N` outside torchrun: run this script under
    torch.distributed.run with N ranks on this node (rendezvous on
    127.0.0.1), NCCL's init log on (the communicator's rank count)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: --gpus {args.gpus} -> {' '.join(cmd[1:6])} ...", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def dist_setup():
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        # gloo = host-side plumbing only (handles, timings, flags); the data
        # path is NCCL or the fused peer kernel
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


def cuda_alive() -> bool:
    """False once this process's CUDA context carries a sticky error."""
    import torch
    try:
        torch.cuda.synchronize()
        return True
    except Exception:  # noqa: BLE001
        traceback.print_exc()
        return False


def all_ok(ok: bool, world: int) -> bool:
    if world == 1:
        return ok
    import torch
    import torch.distributed as dist
    t = torch.tensor([0 if ok else 1], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t[0]) == 0


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


def device_sync(comm, stream, timeout_ms: int):
    """Waits for `stream`; with an NCCL communicator through ptk_comm_wait
    (async-error polling + timeout -> ncclCommAbort -> PtkError) so a hung
    peer fails the leg instead of hanging the job."""
    import torch
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import stream_handle
    if comm is not None:
        nat.lib.ptk_comm_wait(comm, stream_handle(stream), timeout_ms)
    torch.cuda.synchronize()


def traffic_from_profiles(workload):
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def workload_config(args, numels, desc, world) -> dict:
    """The workload description shared by the GPU and the CPU reference arm."""
    return {"workload": f"{args.workload}: {desc}", "params": sum(numels), "chunks": len(numels),
            "chunk_params": numels if len(numels) <= 16 else
            {"n": len(numels), "first": numels[0], "last": numels[-1]},
            "parallelism": f"zero3-dp{world}",
            "l2": "inputs larger than L2 (%.1f GB touched per step per rank)"
                  % (metric_hbm_bytes(numels, world) / 1e9),
            "algorithmic_bytes_per_step_per_rank": metric_hbm_bytes(numels, world),
            "nvlink_bytes_per_step_per_rank": nvlink_bytes(numels, world),
            "bytes_accounting": "BASELINE.md §3 HBM formula, identical for every exchange and arm"}


# ------------------------------------------------------------------ GPU arm --

def run_gpu(args):
    import torch
    from paper_2406_08334_b200 import _native as nat

    world, rank, local = dist_setup()
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.exchange == "auto":
        legs = ["nccl"] if world == 1 else ["nccl", "fused"]
    else:
        legs = [args.exchange]
    if args.shared_device:
        # flow validation on a one-GPU box: every rank on cuda:0, peers mapped
        # through cudaIpc as on an NVLink node; NCCL refuses duplicate devices,
        # so only the fused exchange runs and the timings are not a bench value
        legs = ["fused"]
        local = 0
        args.train_exchange = "fused"   # NCCL refuses two ranks on one device
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numels, desc = chunk_numels(args.workload)
    hbm_peak, peak_kind = load_peaks()

    results = {}
    for mode in legs:
        err = None
        if world > 1:
            # N > 1: each exchange in a guarded child job (run_exchange_child),
            # so a hang or device fault in one leg cannot lose the other
            res, err = run_exchange_child(args, world, rank, local, mode)
        else:
            try:
                res = run_leg(args, mode, numels, world, rank, local, dev, hbm_peak, peak_kind)
            except Exception as e:  # noqa: BLE001  (one failing leg must not lose the line)
                err = f"{type(e).__name__}: {e}"
                traceback.print_exc()
                res = None
        ok = all_ok(err is None, world)
        if ok:
            results[mode] = res
        else:
            results[mode] = {"error": err or "failed on another rank"}
        if not cuda_alive():
            # a sticky device error (e.g. a trapped peer barrier) poisons this
            # context: keep the legs measured so far and touch the GPU no more
            results[mode]["error"] = (results[mode].get("error") or "") + "; CUDA context lost"
            break
        torch.cuda.empty_cache()
    gpu_ok = cuda_alive()
    done = {m: r for m, r in results.items() if "error" not in r}
    if not done:
        raise SystemExit(f"bench.py: every exchange leg failed: {results}")
    best = max(done, key=lambda m: done[m]["value"])
    lead = done[best]

    train = train_offload = None
    if args.train_steps > 0 and args.workload in TRAIN_MODELS and (gpu_ok or world > 1):
        if world == 1:
            train = run_train(args, world, rank, dev, None)
            if args.offload_persist >= 0:
                train_offload = run_train(args, world, rank, dev, None,
                                          n_persist=args.offload_persist,
                                          n_buffer=args.offload_buffers)
        else:
            # N > 1: the NCCL training path runs in guarded child processes
            # (own process group, timeout) so no failure there can lose the
            # chunk-step line
            train = run_train_child(args, world, rank, local, n_persist=-1)
            if args.offload_persist >= 0:
                train_offload = run_train_child(args, world, rank, local,
                                                n_persist=args.offload_persist)
    copy_peak = live_copy_peak() if gpu_ok else None

    result = None
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, numels, world)
    barrier(world)
    if rank == 0:
        roof = dict(lead["roofline"], live_copy_gbs_this_box=copy_peak)
        if roof.get("bound") == "hbm" and copy_peak:
            roof["frac_of_live_copy"] = round(roof["achieved"] / copy_peak, 4)
        result = {
            "metric": METRIC,
            "value": lead["value"],
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": lead["ms_per_step"],
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32 (Adam state) / bf16 (grads, params)",
            "data": "synthetic (counter-based uniform; SURVEY §8(d) seeds)",
            "config": workload_config(args, numels, desc, world),
            "exchange": best if world > 1 else "none (w=1)",
            "exchanges": {m: {k: v for k, v in r.items() if k not in ("e2e",)}
                          for m, r in results.items()},
            "timed_steps": lead["timed_steps"],
            "roofline": roof,
            "e2e": lead.get("e2e"),
            "train": train,
            "train_offload": train_offload,
            "gpu_launches": lead["launches"],
            "clocks": lead["clocks"],
            "grad_stats": lead["grad_stats"],
            "cpu_baseline": cpu,
        }
        if args.shared_device:
            result["shared_device_validation"] = "all ranks on cuda:0: flow check, not a bench value"
    return result


def run_leg(args, mode, numels, world, rank, local, dev, hbm_peak, peak_kind):
    """One exchange: build the rank's chunks, warm up, time K steps (device
    events, barrier + sync on both sides, max over ranks), time the dominant
    kernel per launch, check the gathered chunks agree across ranks, run the
    e2e variant."""
    import torch
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet

    comm = make_comm(world, rank) if (mode == "nccl" and world > 1) else None
    symmetric = comm is not None and args.nccl_symmetric
    cs = ChunkSet(numels, world=world, rank=rank, device=dev, mode=mode, comm=comm,
                  symmetric=symmetric)
    try:
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
        timeout = args.comm_timeout_ms

        for _ in range(args.warmup):
            cs.step(hyper)
        device_sync(comm, stream, timeout)
        barrier(world)

        # N = 1 (--graph): the K timed steps are captured once into a CUDA
        # graph (each step with its own step number, so one replay performs
        # exactly steps n+1..n+K) and the timed region is one replay.
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
            device_sync(comm, stream, timeout)
            barrier(world)
        launches = nat.launch_count() - launches0
        del graph
        ms = max_over_ranks(start.elapsed_time(end) / args.steps, world)
        value = metric_hbm_bytes(numels, world) * world / (ms * 1e-3) / 1e9

        consistent = gathered_consistent(cs, world)   # after the steps' all-gathers
        sumsq, nonfinite = cs.grad_stats()
        kern = time_dominant_kernel(cs, hyper, stream, world, numels,
                                    reps=max(1, min(args.steps, 5)), use_graph=use_graph,
                                    comm=comm, timeout=timeout)
        e2e = run_e2e(cs, hyper, args, world, numels, comm) if not args.no_e2e else None
        # step-level roofline: T* = max(HBM / peak, NVLink / peak) per rank
        hbm_req = required_hbm_bytes(numels, world, mode) if world > 1 else metric_hbm_bytes(numels, 1)
        t_hbm = hbm_req / (hbm_peak * 1e9)
        t_nvl = nvlink_bytes(numels, world) / (NVLINK_GBS * 1e9)
        t_star = max(t_hbm, t_nvl)
        roof = roofline(kern, hbm_peak, peak_kind, args.workload)
        roof["step"] = {"t_star_ms": round(t_star * 1e3, 4), "ms_per_step": round(ms, 4),
                        "frac": round(t_star * 1e3 / ms, 4),
                        "bound": "nvlink" if t_nvl > t_hbm else "hbm",
                        "hbm_bytes_required_per_rank": hbm_req,
                        "nvlink_bytes_per_rank_per_dir": nvlink_bytes(numels, world),
                        "serialized_ms": round((t_hbm + t_nvl) * 1e3, 4)}
        out = {"value": round(value, 2), "ms_per_step": round(ms, 4),
               "timed_steps": ("one CUDA-graph replay holding the K steps" if use_graph
                               else "K host-launched steps"),
               "roofline": roof, "launches": launches, "clocks": clocks.summary(),
               "grad_stats": {"sumsq": sumsq, "nonfinite": nonfinite,
                              "scope": "this rank's shards" if world > 1 else "all chunks"},
               "consistent_across_ranks": consistent, "e2e": e2e,
               "kernel": kern["kernel"]}
        if comm is not None:
            out["nccl_buffers"] = ("NCCL symmetric windows (ncclMemAlloc + ncclCommWindowRegister)"
                                   if symmetric else "cudaMalloc (caching allocator)")
        if not consistent:
            raise RuntimeError("gathered parameter chunks differ across ranks")
        return out
    finally:
        torch.cuda.synchronize()
        barrier(world)   # no rank unmaps / frees while a peer may still store into it
        if mode == "fused" and world > 1:
            cs.close_ipc_peers()
        cs.close()
        del cs
        if comm is not None:
            nat.lib.ptk_comm_destroy(comm)


def gathered_consistent(cs, world) -> bool:
    """After an all-gather every rank holds the same full parameter chunks:
    compare a checksum of the int16 bits of every chunk across ranks."""
    import torch
    if world == 1:
        return True
    import torch.distributed as dist
    piece = 1 << 26
    sums = torch.tensor([sum(int(torch.sum(c.param[lo:lo + piece].view(torch.int16),
                                           dtype=torch.int64))
                             for lo in range(0, c.n_pad, piece)) for c in cs.chunks],
                        dtype=torch.int64)
    allsums = [torch.zeros_like(sums) for _ in range(world)]
    dist.all_gather(allsums, sums)
    return all(torch.equal(allsums[0], s) for s in allsums)


def time_dominant_kernel(cs, hyper, stream, world, numels, reps, use_graph=False, comm=None,
                         timeout=0):
    """Average launch duration of the step's dominant kernel (CUDA events on
    the stream it is launched on) and its algorithmic bytes per launch: the
    chunk-table Adam (w = 1 / nccl) or the fused table kernel, ONE launch per
    step covering every chunk. `reps` launches back to back (a CUDA graph of
    them at N = 1) between two events on the launching stream."""
    import torch
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import stream_handle, vp
    cfg = hyper.config(cs.step_count + 1, world)

    def launch(sh):
        if cs.mode == "fused":
            nat.lib.ptk_fused_step_table(ctypes.byref(cfg), cs.fused_table, vp(cs.stats),
                                         vp(cs.workspace), None, None, sh)
        else:
            nat.lib.ptk_chunk_adam_table(ctypes.byref(cfg), cs.table, vp(cs.stats),
                                         vp(cs.workspace), None, None, sh)

    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if use_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            sh = stream_handle(None)
            for _ in range(reps):
                launch(sh)
        torch.cuda.synchronize()
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        del g
    else:
        sh = stream_handle(stream)
        e0.record(stream)
        for _ in range(reps):
            launch(sh)
        e1.record(stream)
        device_sync(comm, stream, timeout)
    barrier(world)
    ms = e0.elapsed_time(e1)
    hbm, nvl = dominant_kernel_bytes(numels, world, cs.mode)
    if cs.mode == "fused":
        name = f"fused table kernel ({cs.fused_kernel}: " + (
            "fused_peer_tma_kernel" if cs.fused_kernel == "tma" else "fused_peer_kernel") + ")"
    else:
        name = "chunk_adam_tma_kernel, chunk table (" + nat.raw.ptk_adam_kernel_name().decode() + ")"
    return {"kernel": name, "ms": ms, "hbm_bytes": hbm * reps, "nvl_bytes": nvl * reps,
            "launches": reps, "chunks_per_launch": len(numels), "world": world,
            "timing": "graph of back-to-back launches" if use_graph
            else "back-to-back launches between two events"}


def roofline(k, hbm_peak, peak_kind, workload):
    t_hbm = k["hbm_bytes"] / (hbm_peak * 1e9)
    t_nvl = k["nvl_bytes"] / (NVLINK_GBS * 1e9)
    nvl_bound = t_nvl > t_hbm
    sec = k["ms"] * 1e-3
    achieved = (k["nvl_bytes"] if nvl_bound else k["hbm_bytes"]) / sec / 1e9
    peak = NVLINK_GBS if nvl_bound else hbm_peak
    out = {"bound": "nvlink" if nvl_bound else "hbm", "kernel": k["kernel"],
           "achieved": round(achieved, 1), "peak": peak,
           "peak_kind": "measured peer copy per direction (B200_PROFILING.md)" if nvl_bound
           else peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
           "traffic": traffic_from_profiles(workload) if k["world"] == 1 else None,
           "bytes_per_launch": (k["nvl_bytes"] if nvl_bound else k["hbm_bytes"]) // k["launches"],
           "hbm_bytes_per_launch": k["hbm_bytes"] // k["launches"],
           "nvlink_bytes_per_launch": k["nvl_bytes"] // k["launches"],
           "chunks_per_launch": k["chunks_per_launch"],
           "ms_per_launch": round(k["ms"] / k["launches"], 4),
           "launch_timing": k["timing"],
           "frac_of_8tbs_spec": None if nvl_bound else round(achieved / 8000.0, 4)}
    if k["world"] > 1:
        out["hbm_gbs"] = round(k["hbm_bytes"] / sec / 1e9, 1)
        out["nvlink_gbs_per_dir"] = round(k["nvl_bytes"] / sec / 1e9, 1)
    return out


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
    # N > 1: the persistent chunks' step is the fused RS->Adam->AG kernel over
    # NVLink peer memory and the non-persistent chunks (ChunkPool) gather and
    # reduce over peer memory too -- no library collective
    # (--train-exchange nccl: NCCL for both, the library path)
    mode = train_exchange_mode(args, world)
    cs = ChunkSet(numels[:np_], world=world, rank=rank, device=dev, mode=mode,
                  comm=comm if mode == "nccl" else None)
    pool = (ChunkPool(numels, np_, n_buffer, world=world, rank=rank, comm=comm, device=dev,
                      exchange="peer" if mode == "fused" else "nccl")
            if np_ < len(numels) else None)
    shape = GPT2Shape.from_trace(trace)
    model = ChunkedGPT2(shape, layout, cs, trace["ops"], pool=pool)
    model.init_weights(seed=0)
    if mode == "fused":
        cs.attach_ipc_peers()
        if pool is not None:
            pool.attach_ipc_peers()
    batch = int(trace["meta"]["batch_size"])
    n_iter = args.warmup + args.train_steps
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    # learnable synthetic stream (next token = token + 1) so the loss is a sanity signal
    tokens = torch.randint(0, shape.vocab, (n_iter, batch, shape.seq), device=dev, generator=gen)
    targets = (tokens + 1) % shape.vocab
    hyper = AdamHyper(lr=1e-4, weight_decay=0.01, adamw=True)
    stream = torch.cuda.current_stream()
    losses = []
    overlap = args.train_overlap and mode == "nccl"
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
    if world > 1:
        out["exchange"] = ("fused RS->Adam->AG table kernel over NVLink peer memory"
                           + ("; pool: peer all-gather + fp32 peer reduce-scatter"
                              if pool is not None else "")
                           if mode == "fused" else
                           "NCCL RS / AG per chunk (ChunkSet nccl mode, ChunkPool)")
    if pool is not None:
        out["offload"] = {"pinned_host_GB": round(pool.host_bytes / 1e9, 3),
                          "buffer_GB": round(pool.device_bytes / 1e9, 3),
                          "fetches": pool.counters["fetch"], "evictions": pool.counters["evict"],
                          "h2d_GB": round(pool.counters["h2d_bytes"] / 1e9, 2),
                          "d2h_GB": round(pool.counters["d2h_bytes"] / 1e9, 2)}
    if mode == "fused":
        torch.cuda.synchronize()
        barrier(world)   # no rank unmaps while a peer may still store into it
        cs.close_ipc_peers()
        if pool is not None:
            pool.close_ipc_peers()
    del model, cs, pool
    torch.cuda.empty_cache()
    return out


def train_exchange_mode(args, world) -> str:
    return "fused" if world > 1 and args.train_exchange == "fused" else "nccl"


def _run_child(args, world, rank, local, extra, timeout, what, env_extra=None):
    """Runs this script again as one rank of a child job (its own gloo group
    on a fresh port, its own CUDA context, a timeout) and returns
    (result dict or None, error string or None). A failure, hang or device
    fault inside the child is reported instead of losing the bench line."""
    import torch
    import torch.distributed as dist
    port = torch.tensor([free_port() if rank == 0 else 0], dtype=torch.int64)
    dist.broadcast(port, 0)
    fd, out_path = tempfile.mkstemp(prefix=f"ptk_{what}_r{rank}_", suffix=".json")
    os.close(fd)
    # not torchrun's agent store: the child job rendezvouses on its own port
    # (with TORCHELASTIC_USE_AGENT_STORE inherited, every child would wait
    # for a store server that never comes up on that port)
    env = {k: v for k, v in os.environ.items() if not k.startswith("TORCHELASTIC_")}
    env.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(int(port[0])), RANK=str(rank),
               WORLD_SIZE=str(world), LOCAL_RANK=str(local), **(env_extra or {}))
    cmd = [sys.executable, os.path.abspath(__file__)] + sys.argv[1:] + extra + ["--leg-out", out_path]
    barrier(world)
    t0 = time.time()
    try:
        # the child's stdout (NCCL_DEBUG=INFO init lines: "comm ... nRanks N") goes to
        # this rank's stderr: visible to the driver, never mixed into the JSON line
        p = subprocess.run(cmd, env=env, timeout=timeout, stdout=sys.stderr.fileno())
        rc = p.returncode
    except subprocess.TimeoutExpired:
        rc = "timeout"
    res = None
    try:
        with open(out_path) as f:
            res = json.load(f) if rc == 0 else None
    except Exception:  # noqa: BLE001
        res = None
    finally:
        os.unlink(out_path)
    barrier(world)
    if res is None:
        return None, f"{what} child exited with {rc} after {time.time() - t0:.0f} s"
    return res, None


def run_train_child(args, world, rank, local, n_persist):
    """The training leg at N > 1 in a child process per rank: a failure or
    hang there is reported in the line instead of losing it. All-persistent
    training runs the fused exchange first and, if that child fails on any
    rank, is retried with NCCL (the line says so)."""
    extra = ["--leg", "train", "--leg-persist", str(n_persist)]
    res, err = _run_child(args, world, rank, local, extra, args.train_timeout, "train")
    fused_first = train_exchange_mode(args, world) == "fused"
    if all_ok(res is not None, world) or not fused_first or args.shared_device:
        return res if res is not None else {"error": err}
    res, err2 = _run_child(args, world, rank, local, extra + ["--train-exchange", "nccl"],
                           args.train_timeout, "train_nccl")
    if res is not None:
        res["fallback"] = f"fused-exchange training failed ({err}); NCCL"
        return res
    return {"error": f"{err}; NCCL retry: {err2}"}


def run_exchange_child(args, world, rank, local, mode):
    """An exchange leg at N > 1 in a child process per rank. The fused leg
    runs the TMA-ring kernel first; if that child fails on any rank (a device
    fault poisons only the child's context), every rank retries with the
    register-staged kernel (PTK_FUSED_KERNEL=ldg) and the line says so."""
    res, err = _run_child(args, world, rank, local, ["--leg", "exchange", "--leg-mode", mode],
                          args.leg_timeout, f"exchange_{mode}")
    if all_ok(res is not None, world):
        return res, err
    if mode == "nccl" and args.nccl_symmetric:
        # symmetric windows need NCCL/driver support: retry on plain buffers
        first = err or "failed on another rank"
        res, err = _run_child(args, world, rank, local, ["--leg", "exchange", "--leg-mode", mode,
                                                         "--no-nccl-symmetric"],
                              args.leg_timeout, "exchange_nccl_plain")
        if res is not None:
            res["fallback"] = f"NCCL symmetric-window leg failed ({first}); plain buffers"
            return res, None
        return None, f"{first}; plain-buffer retry: {err}"
    if mode != "fused" or os.environ.get("PTK_FUSED_KERNEL"):
        return res, err
    first = err or "failed on another rank"
    res, err = _run_child(args, world, rank, local, ["--leg", "exchange", "--leg-mode", mode],
                          args.leg_timeout, "exchange_fused_ldg", {"PTK_FUSED_KERNEL": "ldg"})
    if res is not None:
        res["fallback"] = f"TMA-ring fused kernel failed ({first}); register-staged kernel"
        return res, None
    return None, f"{first}; ldg retry: {err}"


def run_exchange_leg(args):
    """--leg exchange: the child of run_exchange_child."""
    import torch
    world, rank, local = dist_setup()
    if args.shared_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numels, _ = chunk_numels(args.workload)
    hbm_peak, peak_kind = load_peaks()
    if (os.environ.get("PTK_BENCH_INJECT_FAULT") == "fused-tma"
            and os.environ.get("PTK_FUSED_KERNEL") != "ldg"):   # test hook of the retry path
        raise SystemExit("bench.py: injected fault in the TMA-ring fused leg")
    res = run_leg(args, args.leg_mode, numels, world, rank, local, dev, hbm_peak, peak_kind)
    with open(args.leg_out, "w") as f:
        json.dump(res, f)
    barrier(world)


def run_train_leg(args):
    """--leg train: the child of run_train_child."""
    import torch
    world, rank, local = dist_setup()
    if args.shared_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n_persist = None if args.leg_persist < 0 else args.leg_persist
    fused = train_exchange_mode(args, world) == "fused"
    comm = None if fused else make_comm(world, rank)
    res = run_train(args, world, rank, dev, comm, n_persist=n_persist,
                    n_buffer=args.offload_buffers if n_persist is not None else 0)
    torch.cuda.synchronize()
    with open(args.leg_out, "w") as f:
        json.dump(res, f)
    barrier(world)
    if comm is not None:
        from paper_2406_08334_b200 import _native as nat
        nat.lib.ptk_comm_destroy(comm)


def e2e_pieces(n: int, piece: int, ramp_up: bool, ramp_down: bool, first: int = 1 << 20):
    """(offset, length) pieces covering [0, n): `piece`-sized in the middle,
    doubling from `first` at the start (ramp_up) and halving to `first` at
    the end (ramp_down). Every boundary is a multiple of 8 elements."""
    ramp = []
    k = first
    while k < piece:
        ramp.append(k)
        k *= 2
    head = ramp if ramp_up else []
    tail = ramp[::-1] if ramp_down else []
    if sum(head) + sum(tail) >= n:   # too small to ramp: plain pieces
        head, tail = [], []
    sizes = list(head)
    mid = n - sum(head) - sum(tail)
    sizes += [piece] * (mid // piece)
    if mid % piece:
        sizes.append(mid % piece)
    sizes += tail
    out, lo = [], 0
    for m in sizes:
        out.append((lo, m))
        lo += m
    assert lo == n
    return out


def run_e2e(cs, hyper, args, world, numels, comm):
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
        last = len(cs.chunks) - 1
        for c, hg, hp in zip(cs.chunks, host_g, host_p):
            # at least ~8 pieces per chunk so copies overlap the update even
            # for small chunks (multiple of 12288 elements: whole TMA tiles);
            # the step's first pieces grow and its last ones shrink
            # geometrically, so the pipeline fill (first H2D) and drain (last
            # D2H) cost one small piece instead of one full piece each
            pc = min(piece, max(1 << 20, -(-c.shard // 8 // 12288) * 12288))
            for lo, n in e2e_pieces(c.shard, pc, ramp_up=c.chunk_id == 0,
                                    ramp_down=c.chunk_id == last):
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
    device_sync(comm, comp, args.comm_timeout_ms)
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(comp)
    for _ in range(steps):
        one_step()
    t1.record(comp)
    device_sync(comm, comp, args.comm_timeout_ms)
    barrier(world)
    ms = max_over_ranks(t0.elapsed_time(t1) / steps, world)
    h2d_bytes = sum(2 * span(c) for c in cs.chunks)
    d2h_bytes = sum(2 * span(c) for c in cs.chunks) + 16
    value = metric_hbm_bytes(numels, world) * world / (ms * 1e-3) / 1e9
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
                    ("C-ABI: H2D local grad chunks -> ptk_peer_barrier -> ptk_fused_step_table "
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

def host_mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 16 << 30


class CpuChunkStep:
    """The SAME chunk step on the host through the oracle port
    (oracle/chunk_step.c, OpenMP over every host thread), inputs from the same
    counter-based seeds as the GPU arm. w = 1: fp32 Adam of every chunk with
    its bf16 gradient, bf16 parameters out. w > 1: w simulated ranks per
    chunk -- rank-order fp32 reduce-scatter of the w gradient chunks into the
    owner shard, Adam on each shard (grad scale 1/w), all-gather of the bf16
    shards into every rank's parameter chunk. When the host cannot hold the
    full workload (MemAvailable / 2), every chunk is shortened by one common
    factor (`sample` says so)."""

    def __init__(self, numels, world: int):
        import numpy as np
        sys.path.insert(0, os.path.join(REPO, "tests"))
        import oracle_lib as ol
        from paper_2406_08334_b200.chunks import GRAD_SCALE, MASTER_SCALE, grad_seed, master_seed
        self.ol, self.world = ol, world
        # every host thread (torchrun exports OMP_NUM_THREADS=1 to its ranks)
        ol.set_num_threads(len(os.sched_getaffinity(0)))
        per_param = 16 if world == 1 else 12 + 4 * world + 2 + 4
        budget = host_mem_available() // 2
        need = per_param * sum(numels)
        self.factor = min(1.0, budget / need) if need else 1.0
        self.numels = [max(8 * world, int(n * self.factor)) // (8 * world) * (8 * world)
                       if self.factor < 1.0 else n for n in numels]
        self.chunks = []
        for ci, n in enumerate(self.numels):
            shard = ol.shard_elems(n, world)
            n_pad = shard * world
            master = ol.fill_f32(n_pad, master_seed(ci), MASTER_SCALE)
            master[n:] = 0
            if world == 1:
                g = ol.fill_bf16(n_pad, grad_seed(ci, 0, 0), GRAD_SCALE)
                self.chunks.append(dict(n=n, shard=shard, master=[master], m=[np.zeros(n_pad, np.float32)],
                                        v=[np.zeros(n_pad, np.float32)], grads=[g],
                                        params=[np.zeros(n_pad, np.uint16)]))
                continue
            grads = []
            for q in range(world):
                g = ol.fill_bf16(n_pad, grad_seed(ci, q, 0), GRAD_SCALE)
                g[n:] = 0
                grads.append(g)
            self.chunks.append(dict(
                n=n, shard=shard,
                master=[master[r * shard:(r + 1) * shard].copy() for r in range(world)],
                m=[np.zeros(shard, np.float32) for _ in range(world)],
                v=[np.zeros(shard, np.float32) for _ in range(world)],
                grads=grads, outs=[np.zeros(shard, np.uint16) for _ in range(world)],
                params=[np.zeros(n_pad, np.uint16) for _ in range(world)],
                red=np.zeros(shard, np.float32)))
        self.step_count = 0

    def step(self):
        ol, w = self.ol, self.world
        self.step_count += 1
        s = ol.scalars(lr=1e-3, step=self.step_count, grad_scale=1.0 / w)
        for c in self.chunks:
            if w == 1:
                ol.adam_step(s, c["master"][0], c["m"][0], c["v"][0], c["grads"][0], c["params"][0])
                continue
            arr = (ctypes.c_void_p * w)(*[g.ctypes.data for g in c["grads"]])
            for r in range(w):
                ol.lib.oracle_reduce_scatter_f32(arr, w, r, c["shard"], ol._p(c["red"]))
                ol.adam_step(s, c["master"][r], c["m"][r], c["v"][r], c["red"], c["outs"][r])
            shards = (ctypes.c_void_p * w)(*[o.ctypes.data for o in c["outs"]])
            for r in range(w):
                ol.lib.oracle_allgather_bf16(shards, w, c["shard"], ol._p(c["params"][r]))

    def sample(self) -> str:
        full = "the full workload" if self.factor >= 1.0 else (
            f"every chunk shortened to {self.factor:.3f} of its length (host memory)")
        return (f"oracle port (oracle/chunk_step.c) of the chunk step over {sum(self.numels)} "
                f"params in {len(self.numels)} chunks ({full})"
                + (f", {self.world} simulated ranks (rank-order fp32 RS, Adam per shard, AG)"
                   if self.world > 1 else ", w=1 (Adam, bf16 params out)")
                + "; the reference memplan never executes the data plane (SPEC.md:514)")


def cpu_chunk_step_timing(numels, world, steps, warmup):
    """Times the host chunk step: `warmup` untimed then `steps` timed steps
    (wall clock of the OpenMP kernels). Returns (ms per step, value GB/s,
    runner)."""
    run = CpuChunkStep(numels, world)
    for _ in range(warmup):
        run.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        run.step()
    dt = (time.perf_counter() - t0) / steps
    value = metric_hbm_bytes(run.numels, world) * world / dt / 1e9
    return dt * 1e3, value, run


def cpu_extras(args) -> dict:
    """the reference's own CPU tool on the same
    config (oracle/_ref/memplan plan / simulate wall time, unmodified
    reference build) and torch CPU Adam(fused=True) params/s (the
    calibration point of cpu_optim_rate)."""
    out = {}
    ref = os.path.join(REPO, "oracle", "_ref", "memplan")
    name = TRAIN_MODELS.get(args.workload) or "gpt2-1.5b_b8"
    if os.path.exists(ref):
        try:
            from paper_2406_08334_b200 import planner
            with tempfile.TemporaryDirectory(prefix="ptk_refcpu_") as d:
                trace = os.path.join(d, "trace.json")
                subprocess.run([ref, "gen-trace"] + planner.TRACE_ARGS[name] + ["-o", trace],
                               check=True, capture_output=True, timeout=120)
                hw = ["--hw", "a100x1", "--gpu-mem", "180000000000", "--coll-bw", "9e11",
                      "--h2d-bw", "5.5e10", "--d2h-bw", "5.5e10", "--cpu-mem", "2000000000000",
                      "--gpu-optim-rate", "2e11", "--world-size", "1"]
                for verb, extra in (("plan", []), ("simulate", ["--n-persist", "3"])):
                    t0 = time.perf_counter()
                    subprocess.run([ref, verb, "--trace", trace] + hw + extra, check=True,
                                   capture_output=True, timeout=300)
                    out[f"memplan_{verb}_s"] = round(time.perf_counter() - t0, 4)
            out["memplan"] = f"oracle/_ref/memplan (reference, unmodified) on {name}, B200-like flags"
        except Exception as e:  # noqa: BLE001
            out["memplan_error"] = repr(e)
    else:
        out["memplan_error"] = "oracle/_ref/memplan not built"
    try:
        import torch
        torch.set_num_threads(len(os.sched_getaffinity(0)))
        n = 64 * 1024 * 1024
        p = torch.nn.Parameter(torch.randn(n) * 0.05)
        p.grad = torch.randn(n) * 1e-3
        opt = torch.optim.Adam([p], lr=1e-3, fused=True)
        opt.step()
        t0 = time.perf_counter()
        for _ in range(3):
            opt.step()
        dt = (time.perf_counter() - t0) / 3
        out["torch_cpu_fused_adam_params_per_s"] = round(n / dt, 1)
        out["torch_cpu_fused_adam_threads"] = torch.get_num_threads()
        del p, opt
    except Exception as e:  # noqa: BLE001
        out["torch_cpu_adam_error"] = repr(e)
    return out


def cpu_baseline(args, numels, world):
    """In-run CPU baseline (rank 0): the same host chunk step as the
    reference arm, 1 warm-up + 3 timed steps, plus the BASELINE.md §2 extras."""
    ms, value, run = cpu_chunk_step_timing(numels, world, steps=3, warmup=1)
    out = {"value": round(value, 3), "unit": "GB/s", "cores": run.ol.num_threads(), "kind": "port",
           "ms_per_step": round(ms, 2), "sample": run.sample() + "; 1 warm-up + 3 timed steps",
           "same_config": run.factor >= 1.0}
    del run
    out["extras"] = cpu_extras(args)
    return out


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path on
    this box's host cores (the oracle port: the reference never executes
    the data plane), same workload / metric / unit, rank 0 only."""
    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    numels, desc = chunk_numels(args.workload)
    ms, value, run = cpu_chunk_step_timing(numels, world, steps=args.steps, warmup=args.warmup)
    cpu = {"value": round(value, 3), "unit": "GB/s", "cores": run.ol.num_threads(), "kind": "port",
           "ms_per_step": round(ms, 2),
           "sample": run.sample() + f"; {args.warmup} warm-up + {args.steps} timed steps",
           "same_config": run.factor >= 1.0}
    same = run.factor >= 1.0
    del run
    cpu["extras"] = cpu_extras(args)
    return {"impl": "reference", "metric": METRIC,
            "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (Adam state) / bf16 (grads, params)",
            "data": "synthetic (counter-based uniform; SURVEY §8(d) seeds)",
            "config": workload_config(args, numels, desc, world),
            "same_config": same,
            "cpu_baseline": cpu,
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
                    help="N>1 chunk exchange: auto = measure both the fused RS->Adam->AG kernel "
                         "over NVLink peer memory and NCCL RS/AG + chunk-table Adam, report the "
                         "faster as `value` (both in `exchanges`)")
    ap.add_argument("--comm-timeout-ms", type=int, default=120_000,
                    help="NCCL legs: abort the communicator when a sync waits longer")
    ap.add_argument("--e2e-piece", type=int, default=32 * 1024 * 1024)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--offload-persist", type=int, default=1,
                    help="also time training with chunks >= this index non-persistent "
                         "(pinned host + host Adam); -1 = skip")
    ap.add_argument("--offload-buffers", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--train-steps", type=int, default=10,
                    help="timed iterations of the end-to-end cfg2 training step (tokens/s); 0 = skip")
    ap.add_argument("--train-timeout", type=int, default=300,
                    help="N>1: seconds before a training child process is killed")
    ap.add_argument("--train-exchange", default="fused", choices=["fused", "nccl"],
                    help="N>1 training: the fused RS->Adam->AG kernel over NVLink peer memory "
                         "for persistent chunks + peer all-gather / fp32 peer reduce-scatter for "
                         "the offloaded pool (default, NCCL retry on failure), or NCCL for both")
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
    ap.add_argument("--nccl-symmetric", action=argparse.BooleanOptionalAction, default=True,
                    help="N>1 NCCL leg: chunk buffers in NCCL symmetric windows (ncclMemAlloc + "
                         "ncclCommWindowRegister), retried on plain buffers if that fails")
    ap.add_argument("--leg-timeout", type=int, default=420,
                    help="N>1: seconds before a fused-exchange child process is killed")
    ap.add_argument("--leg", default=None, choices=[None, "train", "exchange", "ping"],
                    help=argparse.SUPPRESS)
    ap.add_argument("--leg-mode", default="fused", help=argparse.SUPPRESS)
    ap.add_argument("--leg-out", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--leg-persist", type=int, default=-1, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.leg == "train":
        run_train_leg(args)
        return
    if args.leg == "exchange":
        run_exchange_leg(args)
        return
    if args.leg == "ping":   # the child-job mechanism alone (CPU test)
        world, rank, _ = dist_setup()
        barrier(world)
        with open(args.leg_out, "w") as f:
            json.dump({"rank": rank, "world": world}, f)
        return
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        sys.exit(self_launch(args))
    if world_env is not None and int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}: launch with "
                         f"--nproc-per-node {args.gpus}, or without torchrun to self-launch")
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
