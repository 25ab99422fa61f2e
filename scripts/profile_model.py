#!/usr/bin/env python3
"""Close the loop on one B200 (profiler re-feed with measured device timings):

  1. profile the cfg2 training model (GPT-2 1.5B, b8, s1024, params in chunk
     buffers) -> a MEASURED ModelTrace (paper_2406_08334_b200.profiler);
  2. measure the HardwareProfile (ptk_measure_profile);
  3. plan with the planner on measured trace + measured profile;
  4. time the real training iteration (train_step) and execute the plan with
     the chunk runtime replaying the measured op times; report
     real vs runtime vs cost-model iteration time.

Writes gpurun_out/trace_gpt2-1.5b_b8_measured.json, gpurun_out/profile_model.json.
"""
import json
import os
import subprocess
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
OUT = os.path.join(REPO, "gpurun_out")
MEMPLAN = os.path.join(REPO, "build", "memplan")


def main():
    from paper_2406_08334_b200 import planner, runtime
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.profiler import profile_trace
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step
    os.makedirs(OUT, exist_ok=True)
    dev = torch.device("cuda", 0)
    trace = planner.trace_for("gpt2-1.5b_b8")
    layout = planner.layout_for("gpt2-1.5b_b8")
    cs = ChunkSet([c["used_bytes"] // 2 for c in layout["chunks"]], device=dev)
    shape = GPT2Shape.from_trace(trace)
    model = ChunkedGPT2(shape, layout, cs, trace["ops"])
    model.init_weights(0)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randint(0, shape.vocab, (8, shape.seq), device=dev, generator=g)
    y = (x + 1) % shape.vocab
    measured = profile_trace(model, x, y, reps=3)
    tpath = os.path.join(OUT, "trace_gpt2-1.5b_b8_measured.json")
    json.dump(measured, open(tpath, "w"), indent=1)

    # real iteration time
    hyper = AdamHyper(lr=1e-4)
    for _ in range(3):
        train_step(model, x, y, hyper)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        train_step(model, x, y, hyper)
    e1.record()
    torch.cuda.synchronize()
    real = e0.elapsed_time(e1) / 5 * 1e-3
    del model, cs
    torch.cuda.empty_cache()

    base = os.path.join(OUT, "base_profile.json")
    json.dump({"h2d_bw": 5.5e10, "d2h_bw": 5.5e10, "coll_alpha": 2e-5, "coll_bw": 7.7e11,
               "world_size": 1, "gpu_mem": 180_000_000_000, "cpu_mem": 1_000_000_000_000,
               "cpu_optim_rate": 1e9, "gpu_optim_rate": 1e11}, open(base, "w"))
    prof = os.path.join(OUT, "b200x1_measured.json")
    hw = runtime.measure_profile(base, prof)
    plan = json.loads(subprocess.run([MEMPLAN, "plan", "--trace", tpath, "--hw", prof],
                                     check=True, capture_output=True, text=True).stdout)
    ppath = os.path.join(OUT, "plan_measured.json")
    json.dump(plan, open(ppath, "w"), indent=1)
    res = runtime.execute_plan(tpath, ppath, prof, compute_scale=1.0, iterations=3)
    fwd = sum(o["t_fwd"] for o in measured["ops"])
    bwd = sum(o["t_bwd"] for o in measured["ops"])
    row = {"real_train_step_s": real, "runtime_measured_t_iter_s": res["t_iter"],
           "cost_model_t_iter_s": plan["estimate"]["t_iter"], "plan": plan["config"],
           "trace_fwd_s": fwd, "trace_bwd_s": bwd,
           "trace_act_bytes": sum(o["act_bytes"] for o in measured["ops"]),
           "m_fwd": measured["m_fwd"], "measured_profile": hw,
           "tokens_per_s_real": 8 * 1024 / real}
    # 5. a memory-constrained plan (the search must offload / swap / checkpoint),
    #    trained for real with exactly that plan, vs the cost model's estimate
    rows = [row]
    for budget, refine in ((40e9, 0), (40e9, 16), (30e9, 0), (30e9, 16)):
        cplan = json.loads(subprocess.run(
            [MEMPLAN, "plan", "--trace", tpath, "--hw", prof, "--gpu-mem", str(int(budget))] +
            (["--refine-sim", str(refine)] if refine else []),
            check=True, capture_output=True, text=True).stdout)
        cfg = cplan["config"]
        cpath = os.path.join(OUT, f"plan_measured_{int(budget / 1e9)}GB{'_refined' if refine else ''}.json")
        json.dump(cplan, open(cpath, "w"), indent=1)
        sim = json.loads(subprocess.run([MEMPLAN, "simulate", "--trace", tpath, "--hw", prof,
                                         "--plan", cpath], check=True, capture_output=True,
                                        text=True).stdout)
        real_c, info = train_with_plan(cfg, cplan["strategies"], x, y)
        info["simulator_t_iter_s"] = sim["t_iter"]
        info["simulator_m_peak"] = sim["m_peak"]
        rows.append({"gpu_mem_budget": budget, "refine_sim": refine, "plan": cfg,
                     "strategies": "".join(s[0] for s in cplan["strategies"]),
                     "cost_model_t_iter_s": cplan["estimate"]["t_iter"],
                     "cost_model_m_peak": cplan["estimate"]["m_peak"],
                     "real_train_step_s": real_c,
                     "rel_err": abs(real_c - cplan["estimate"]["t_iter"]) / real_c,
                     "tokens_per_s_real": 8 * 1024 / real_c, **info})
    print(json.dumps(rows, indent=1))
    json.dump(rows, open(os.path.join(OUT, "profile_model.json"), "w"), indent=1)


def train_with_plan(cfg, strategies, x, y, iters=5):
    """Train the cfg2 model with a planner config: first n_persist chunks on
    the device, the rest pooled in n_buffer slots, the block schedule."""
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step
    dev = x.device
    trace = planner.trace_for("gpt2-1.5b_b8")
    layout = planner.layout_for("gpt2-1.5b_b8")
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
    np_ = cfg["n_persist"]
    cs = ChunkSet(numels[:np_], device=dev)
    pool = ChunkPool(numels, np_, cfg["n_buffer"], device=dev) if np_ < len(numels) else None
    shape = GPT2Shape.from_trace(trace)
    model = ChunkedGPT2(shape, layout, cs, trace["ops"], pool=pool)
    model.init_weights(0)
    model.set_block_schedule(strategies)
    hyper = AdamHyper(lr=1e-4)
    torch.cuda.reset_peak_memory_stats()
    for _ in range(2):
        train_step(model, x, y, hyper)
    if pool is not None:
        pool.finish_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if pool is not None:
        pool.counters.update(host_wait_s=0.0, host_adam_s=0.0)
    e0.record()
    for _ in range(iters):
        train_step(model, x, y, hyper)
    if pool is not None:
        pool.finish_step()
    e1.record()
    torch.cuda.synchronize()
    counters = dict(pool.counters) if pool is not None else None
    phase = {"fwd": 0.0, "bwd": 0.0, "step": 0.0}
    for _ in range(iters):
        # diagnosis only (synchronised): train_step phase by phase
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        if pool is not None:
            pool.begin_step(model.chunks.step_count + 1, hyper, model.pool_uses())
        loss = model.loss(x, y)
        ev[1].record()
        loss.backward()
        ev[2].record()
        model.chunks.step(hyper)
        ev[3].record()
        torch.cuda.synchronize()
        phase["fwd"] += ev[0].elapsed_time(ev[1]) / iters
        phase["bwd"] += ev[1].elapsed_time(ev[2]) / iters
        phase["step"] += ev[2].elapsed_time(ev[3]) / iters
    if pool is not None:
        pool.finish_step()
    info = {"device_peak_allocated_GB": torch.cuda.max_memory_allocated() / 1e9,
            "phase_ms_synchronised": {k: round(v, 2) for k, v in phase.items()}}
    if counters is not None:
        info["pool"] = counters
    del model, cs, pool
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / iters * 1e-3, info


if __name__ == "__main__":
    main()
