#!/usr/bin/env python3
"""BASELINE configs 3 and 4 end to end on one B200: train a model that does
NOT fit on the device as all-persistent chunks (GPT-2 10B b8, Llama-2 13B b8)
with exactly the plan the cost-model search picks from MEASURED inputs.

  1. profile a K-block model of the same shape (same hidden / heads / ffn /
     vocab, all chunks persistent) with the live profiler -> per-operator
     measured times, saved activations and transient peaks;
  2. the full-depth trace = the synthesized trace's operator list and
     parameter bytes (proj/src/trace.cpp:260-344) with the measured values
     (block operators: median over the profiled blocks; every block of these
     models is identical);
  3. measure the HardwareProfile (ptk_measure_profile);
  4. `memplan plan` on measured trace + measured profile -> (np, nb, ns, nc);
     `memplan simulate` on the same inputs;
  5. train with that plan (persistent chunks in HBM, the rest in pinned host
     memory behind n_buffer device slots with host Adam, swap / checkpoint
     blocks) and report tokens/s, measured iteration time against the
     estimate and the simulation, and the device peak against the model's.

    python scripts/train_large.py --model llama-13b --batch 8
        [--chunk-bytes used,reference,used:refine] [--timeline] [--no-isolate]
Writes gpurun_out/train_large_<model>_b<batch>.json (one row per --chunk-bytes mode).
Each row also carries the simulation under the measured host-memory bandwidth
(`memplan simulate --host-mem-bw`); ":refine" plans with --refine-sim under
it; --timeline records a measured iteration in the simulator's event schema;
every training attempt runs in its own child process (a failed attempt gives
all device and pinned host memory back) and an OOM re-plans with a smaller
device budget.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import tempfile
import time

# Plans fill HBM to within a few GB: let the caching allocator grow segments
# in place instead of fragmenting (set before torch initialises CUDA).
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

import torch  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
OUT = os.path.join(REPO, "gpurun_out")


def memplan(*args) -> dict:
    """One planner command, in process (libptk.so's memplan::run_cli)."""
    from paper_2406_08334_b200 import planner
    return json.loads(planner.run_memplan([str(a) for a in args]))


def spec_of(shape, n_blocks: int) -> dict:
    return {"hidden_size": shape.hidden, "n_blocks": n_blocks, "n_heads": shape.heads,
            "n_kv_heads": shape.kv_heads or shape.heads, "ffn_hidden": shape.ffn_dim,
            "vocab_size": shape.vocab, "seq_len": shape.seq, "gated_mlp": shape.gated,
            "bias": shape.bias, "tied_embeddings": shape.tied,
            "learned_pos_embedding": shape.learned_pos}


def host_available_bytes() -> int:
    avail = None
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable:"):
                avail = int(line.split()[1]) * 1024
    try:
        with open("/sys/fs/cgroup/memory.max") as f:
            lim = f.read().strip()
        if lim != "max":
            with open("/sys/fs/cgroup/memory.current") as f:
                avail = min(avail, int(lim) - int(f.read().strip()))
    except OSError:
        pass
    return avail


def measured_full_trace(full: dict, shape, batch: int, k_blocks: int, dev, work: str) -> dict:
    """Steps 1-2: profile a k-block model of the same shape, expand to full depth."""
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import ChunkSet
    from paper_2406_08334_b200.profiler import profile_trace
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape
    spath = os.path.join(work, "spec_small.json")
    json.dump(spec_of(shape, k_blocks), open(spath, "w"))
    tpath = planner.trace_file(["--spec", spath, "--batch", str(batch)],
                               os.path.join(work, "trace_small.json"))
    small = json.load(open(tpath))
    lay = planner.pack(tpath)
    cs = ChunkSet([c["used_bytes"] // 2 for c in lay["chunks"]], device=dev)
    sshape = GPT2Shape.from_trace(small)
    model = ChunkedGPT2(sshape, lay, cs, small["ops"])
    model.init_weights(0)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randint(0, shape.vocab, (batch, shape.seq), device=dev, generator=g)
    meas = profile_trace(model, x, (x + 1) % shape.vocab, reps=3)
    del model, cs
    torch.cuda.empty_cache()
    return expand_trace(full, meas, k_blocks, torch.cuda.get_device_name())


def expand_trace(full: dict, meas: dict, k_blocks: int, device: str) -> dict:
    """Full-depth measured trace: `full`'s operators and parameter bytes, the
    measured t_fwd / t_bwd / act_bytes / d_peak_op of `meas` (a k-block model
    of the same shape) -- top-level operators one to one, block operators the
    median over the profiled blocks."""
    by_kind: dict[str, list[dict]] = {}
    top: dict[str, dict] = {}
    for o in meas["ops"]:
        if o["block_id"] is None:
            top[o["name"]] = o
        else:
            by_kind.setdefault(o["name"].split(".")[0], []).append(o)
    keys = ("t_fwd", "t_bwd", "act_bytes", "d_peak_op")
    ops = []
    for o in full["ops"]:
        if o["block_id"] is None:
            src = {k: top[o["name"]][k] for k in keys}
        else:
            group = by_kind[o["name"].split(".")[0]]
            src = {k: statistics.median(m[k] for m in group) for k in keys}
            src["act_bytes"] = int(src["act_bytes"])
            src["d_peak_op"] = int(src["d_peak_op"])
        ops.append(dict(o, **src, d_cur_prior=0, d_peak_prior=0, d_cur_op=0))
    meta = dict(full["meta"], generator=f"profile_trace on a {k_blocks}-block model of the same "
                "shape, block operators replicated (median over profiled blocks)",
                timings="measured", device=device)
    return {"meta": meta, "m_fwd": meas["m_fwd"], "n_blocks": full["n_blocks"], "ops": ops}


def phase_split(model, cs, pool, x, y, hyper, iters: int) -> dict:
    """Diagnosis only (synchronised, after the timed run): forward, backward
    and persistent-chunk step of train_step, each bracketed by a device sync,
    plus the host wait for pending host Adam inside forward."""
    acc = {"fwd": 0.0, "bwd": 0.0, "step": 0.0, "host_drain_wait": 0.0}
    for _ in range(iters):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        ev[0].record()
        if pool is not None:
            pool.begin_step(cs.step_count + 1, hyper, model.pool_uses())
        loss = model.loss(x, y)
        ev[1].record()
        loss.backward()
        ev[2].record()
        cs.step(hyper)
        ev[3].record()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if pool is not None:
            pool.finish_step()   # host Adam still running after the device work
        acc["host_drain_wait"] += (time.perf_counter() - t0) * 1e3 / iters
        acc["fwd"] += ev[0].elapsed_time(ev[1]) / iters
        acc["bwd"] += ev[1].elapsed_time(ev[2]) / iters
        acc["step"] += ev[2].elapsed_time(ev[3]) / iters
    return {k: round(v, 2) for k, v in acc.items()}


def record_timeline(model, cs, pool, x, y, hyper, path: str, iters: int = 2) -> dict:
    """`iters` more back-to-back iterations with the measured timeline on
    (simulator schema, paper_2406_08334_b200.timeline; an `iter_start` event
    marks each), written as CSV; returns the summary of the LAST one (steady
    state: the previous iteration's host Adam overlaps it, as in training)."""
    from paper_2406_08334_b200.timeline import (Timeline, summarize, write_chrome_trace,
                                                write_csv)
    from paper_2406_08334_b200.train import train_step
    tl = Timeline()
    model.timeline = cs.timeline = tl
    if pool is not None:
        pool.timeline = tl
    if getattr(model, "_swap", None) is not None:
        model._swap.timeline = tl
    tl.begin()
    for i in range(iters):
        tl.gpu(None, "gpu", "iter_start", f"iter={i}")
        train_step(model, x, y, hyper)
    if pool is not None:
        pool.finish_step()
    rows = tl.end()
    model.timeline = cs.timeline = None
    if pool is not None:
        pool.timeline = None
    if getattr(model, "_swap", None) is not None:
        model._swap.timeline = None
    write_csv(rows, path)
    write_chrome_trace(rows, path[:-4] + ".chrome.json")   # chrome://tracing, simulator layout
    from paper_2406_08334_b200.timeline import last_iteration
    return {"iterations": iters, "last_iteration": summarize(last_iteration(rows))}


def _train_child(full, layout, plan, batch, iters, warmup, phases, timeline_path) -> dict:
    """One training attempt (run in a spawned child with --isolate)."""
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    try:
        return train_with_plan(full, layout, plan, batch, dev, iters, warmup, phases,
                               timeline_path)
    except torch.OutOfMemoryError as e:
        return {"oom": str(e)[:300]}


def train_with_plan(full: dict, layout: dict, plan: dict, batch: int, dev, iters: int,
                    warmup: int, phases: int = 0, timeline_path: str = "") -> dict:
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step
    cfg = plan["config"]
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
    np_ = cfg["n_persist"]
    t0 = time.perf_counter()
    cs = ChunkSet(numels[:np_], device=dev)
    pool = ChunkPool(numels, np_, cfg["n_buffer"], device=dev) if np_ < len(numels) else None
    shape = GPT2Shape.from_trace(full)
    model = ChunkedGPT2(shape, layout, cs, full["ops"], pool=pool)
    model.init_weights(0)
    model.set_block_schedule(plan["strategies"])
    setup_s = time.perf_counter() - t0
    hyper = AdamHyper(lr=1e-4)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randint(0, shape.vocab, (batch, shape.seq), device=dev, generator=g)
    y = (x + 1) % shape.vocab
    losses = []
    torch.cuda.reset_peak_memory_stats()
    torch.cuda.reset_accumulated_memory_stats()
    for _ in range(warmup):
        losses.append(train_step(model, x, y, hyper))
    if pool is not None:
        pool.finish_step()
        pool.counters.update(host_wait_s=0.0, host_adam_s=0.0, fetch=0, evict=0, h2d_bytes=0,
                             d2h_bytes=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for _ in range(iters):
        losses.append(train_step(model, x, y, hyper))
    if pool is not None:
        pool.finish_step()
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) / iters
    t_iter = e0.elapsed_time(e1) / iters * 1e-3
    out = {"t_iter_s": t_iter, "wall_iter_s": wall, "tokens_per_s": batch * shape.seq / t_iter,
           "iters": iters, "warmup": warmup, "setup_s": round(setup_s, 1),
           "losses": [round(float(v), 4) for v in losses],
           "device_peak_allocated_GB": torch.cuda.max_memory_allocated() / 1e9,
           "device_peak_reserved_GB": torch.cuda.max_memory_reserved() / 1e9,
           "alloc_retries": torch.cuda.memory_stats().get("num_alloc_retries", 0),
           "alloc_conf": os.environ.get("PYTORCH_CUDA_ALLOC_CONF", ""),
           "persistent_chunk_GB": sum(16 * c.shard for c in cs.chunks) / 1e9}
    if pool is not None:
        out["pool"] = {k: (round(v, 3) if isinstance(v, float) else v)
                       for k, v in pool.counters.items()}
        out["pool"]["per_iter_h2d_GB"] = pool.counters["h2d_bytes"] / iters / 1e9
        out["pool"]["per_iter_d2h_GB"] = pool.counters["d2h_bytes"] / iters / 1e9
        out["pinned_host_GB"] = pool.host_bytes / 1e9
        out["buffer_GB"] = pool.device_bytes / 1e9
    if phases:
        out["phase_ms_synchronised"] = phase_split(model, cs, pool, x, y, hyper, phases)
    if timeline_path:
        out["timeline"] = {"csv": os.path.basename(timeline_path),
                           **record_timeline(model, cs, pool, x, y, hyper, timeline_path)}
    del model, cs, pool
    release_memory()
    return out


def release_memory() -> None:
    """Give device memory AND pinned host memory back: torch's caching host
    allocator keeps freed pinned blocks (the pool's shards) otherwise."""
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch._C._host_emptyCache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-13b")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--profile-blocks", type=int, default=4)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--host-frac", type=float, default=0.7,
                    help="refuse a plan whose pinned host bytes exceed this fraction of the "
                         "host memory available now (protects the box)")
    ap.add_argument("--gpu-mem", type=int, default=0, help="device budget override (bytes)")
    ap.add_argument("--gpu-mem-margin", type=int, default=10_000_000_000,
                    help="bytes kept free below the allocatable device memory for the "
                         "caching allocator's slack (ignored with --gpu-mem)")
    ap.add_argument("--chunk-bytes", default="used,reference",
                    help="comma list of planner chunk-state accountings to plan + train with "
                         "(reference = 8*s_chunk per persistent chunk; used = 8*used bytes)")
    ap.add_argument("--oom-retries", type=int, default=2,
                    help="on a device OOM, re-plan with the budget lowered by --oom-step")
    ap.add_argument("--oom-step", type=int, default=4_000_000_000)
    ap.add_argument("--isolate", action=argparse.BooleanOptionalAction, default=True,
                    help="train each attempt in a spawned child process (default), so a failed "
                         "attempt releases all device and pinned host memory")
    ap.add_argument("--refine-k", type=int, default=16,
                    help="candidates simulated for a ':refine' accounting (memplan --refine-sim)")
    ap.add_argument("--trace-in", default="", help="use this measured trace instead of profiling")
    ap.add_argument("--profile-in", default="", help="use this HardwareProfile instead of measuring")
    ap.add_argument("--tag", default="", help="suffix of the output file names")
    ap.add_argument("--timeline", action="store_true",
                    help="record one more iteration's measured timeline (simulator schema) and "
                         "summarise it beside the simulator's timeline of the same plan")
    ap.add_argument("--phases", type=int, default=2,
                    help="after timing, this many synchronised iterations split into "
                         "forward / backward / step / host-drain wait (diagnosis)")
    args = ap.parse_args()
    from paper_2406_08334_b200 import planner, runtime
    from paper_2406_08334_b200.train import GPT2Shape
    os.makedirs(OUT, exist_ok=True)
    dev = torch.device("cuda", 0)
    tag = f"{args.model}_b{args.batch}{args.tag}"
    work = tempfile.mkdtemp(prefix="train_large_")
    full_path = planner.trace_file(["--model", args.model, "--batch", str(args.batch)],
                                   os.path.join(work, "trace_synth.json"))
    synth = json.load(open(full_path))
    shape = GPT2Shape.from_trace(synth)
    t0 = time.perf_counter()
    if args.trace_in:   # reuse a measured trace (A/B runs of the runtime on one plan)
        full = json.load(open(args.trace_in))
    else:
        full = measured_full_trace(synth, shape, args.batch, args.profile_blocks, dev, work)
    profile_s = time.perf_counter() - t0
    tpath = os.path.join(OUT, f"trace_{tag}_measured.json")
    json.dump(full, open(tpath, "w"), indent=1)

    base = os.path.join(work, "base_profile.json")
    json.dump({"h2d_bw": 5.5e10, "d2h_bw": 5.5e10, "coll_alpha": 2e-5, "coll_bw": 7.7e11,
               "world_size": 1, "gpu_mem": 180_000_000_000, "cpu_mem": 1_000_000_000_000,
               "cpu_optim_rate": 1e9, "gpu_optim_rate": 1e11}, open(base, "w"))
    prof = os.path.join(OUT, f"profile_{tag}.json")
    if args.profile_in:
        hw = json.load(open(args.profile_in))
        json.dump(hw, open(prof, "w"))
    else:
        hw = runtime.measure_profile(base, prof)
    host_bw = runtime.host_memory_bw()   # for the simulator's host-memory extension
    layout = planner.pack(tpath)
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
    common = {"model": args.model, "batch": args.batch, "seq": shape.seq, "n_gpus": 1,
              "params": sum(numels), "trace_fwd_s": sum(o["t_fwd"] for o in full["ops"]),
              "trace_bwd_s": sum(o["t_bwd"] for o in full["ops"]),
              "profile_s": round(profile_s, 1), "measured_profile": hw}
    rows = []
    for spec in args.chunk_bytes.split(","):
        # "used" / "reference", optionally ":refine" = plan with --refine-sim
        # under the measured host-memory bandwidth (the simulator picks)
        mode, _, refine = spec.partition(":")
        label = spec.replace(":", "_")
        # the device budget is what this process can still allocate (the
        # profile's gpu_mem is the device total, incl. context + workspaces)
        release_memory()
        free_now = torch.cuda.mem_get_info()[0] + torch.cuda.memory_reserved()
        # minus the caching allocator's slack: plans that fill HBM to the last
        # GB made it flush its cache mid-iteration (alloc retries, ~1 s stalls
        # seen in the measured timeline)
        budget = args.gpu_mem or min(hw["gpu_mem"], free_now) - args.gpu_mem_margin
        attempts = []
        for attempt in range(args.oom_retries + 1):
            row = dict(common, chunk_bytes=spec, gpu_mem_budget=budget)
            acct = ["--chunk-bytes", mode, "--gpu-mem", budget]
            extra = (["--refine-sim", args.refine_k, "--host-mem-bw", host_bw]
                     if refine == "refine" else [])
            plan = memplan("plan", "--trace", tpath, "--hw", prof, *acct, *extra)
            ppath = os.path.join(OUT, f"plan_{tag}_{label}.json")
            json.dump(plan, open(ppath, "w"), indent=1)
            sim_tl = os.path.join(OUT, f"sim_timeline_{tag}_{label}.csv")
            sim = memplan("simulate", "--trace", tpath, "--hw", prof, "--plan", ppath, *acct,
                          "--timeline-csv", sim_tl)
            sim_hm = memplan("simulate", "--trace", tpath, "--hw", prof, "--plan", ppath, *acct,
                             "--host-mem-bw", host_bw)
            cfg = plan["config"]
            pinned = 16 * sum(numels[cfg["n_persist"]:])
            swap_act = sum(o["act_bytes"] for o in full["ops"] if o["block_id"] is not None
                           and plan["strategies"][o["block_id"]] == "swap")
            avail = host_available_bytes()
            row.update({"plan": cfg, "strategies": "".join(s[0] for s in plan["strategies"]),
                        "cost_model_t_iter_s": plan["estimate"]["t_iter"],
                        "cost_model_m_peak_GB": plan["estimate"]["m_peak"] / 1e9,
                        "simulator_t_iter_s": sim["t_iter"],
                        "simulator_m_peak_GB": sim["m_peak"] / 1e9,
                        "host_mem_bw_GBs": host_bw / 1e9,
                        "simulator_host_mem_t_iter_s": sim_hm["t_iter"],
                        "pinned_host_needed_GB": (pinned + swap_act) / 1e9,
                        "host_available_GB": avail / 1e9})
            print(json.dumps(row), flush=True)
            if pinned + swap_act > args.host_frac * avail:
                row["skipped"] = (f"plan needs {(pinned + swap_act) / 1e9:.1f} GB pinned host "
                                  f"memory, more than {args.host_frac} x {avail / 1e9:.1f} GB")
                break
            tl_path = os.path.join(OUT, f"timeline_{tag}_{label}.csv") if args.timeline else ""
            job = (full, layout, plan, args.batch, args.iters, args.warmup, args.phases, tl_path)
            if args.isolate:
                # a child process per attempt: an OOM (or any failure) gives
                # every device and pinned host byte back when the child exits
                release_memory()
                import multiprocessing as mp
                with mp.get_context("spawn").Pool(1) as workers:
                    res = workers.apply(_train_child, job)
            else:
                res = _train_child(*job)
            if "oom" in res:
                attempts.append({"gpu_mem_budget": budget, "plan": cfg, "oom": res["oom"]})
                release_memory()
                budget -= args.oom_step
                continue
            row.update(res)
            if args.timeline:
                from paper_2406_08334_b200.timeline import read_csv, summarize
                row["simulated_timeline"] = {"csv": os.path.basename(sim_tl),
                                             **summarize(read_csv(sim_tl))}
            row["rel_err_cost_model"] = abs(res["t_iter_s"] - row["cost_model_t_iter_s"]) / res["t_iter_s"]
            row["rel_err_simulator"] = abs(res["t_iter_s"] - row["simulator_t_iter_s"]) / res["t_iter_s"]
            row["rel_err_simulator_host_mem"] = (abs(res["t_iter_s"] - row["simulator_host_mem_t_iter_s"])
                                                 / res["t_iter_s"])
            break
        row["oom_attempts"] = attempts
        rows.append(row)
        print(json.dumps(row, indent=1), flush=True)
    json.dump(rows, open(os.path.join(OUT, f"train_large_{tag}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
