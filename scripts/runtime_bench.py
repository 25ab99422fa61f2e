#!/usr/bin/env python3
"""Profiler re-feed + chunk-runtime measurement on one B200.

1. measure this machine's HardwareProfile (ptk_measure_profile): pinned
   H2D/D2H bandwidth, fused chunk Adam and host Adam rates, memory sizes;
2. for each case, plan with the planner under the MEASURED profile
   (`memplan plan --hw measured.json`, or a forced config), execute the plan
   with the chunk runtime (real uploads/offloads/NCCL/device+host Adam,
   stand-in compute of the trace's op times) and compare the measured
   iteration with the cost model's estimate.

Writes gpurun_out/runtime_bench.jsonl and gpurun_out/b200x1_measured.json.
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
OUT = os.path.join(REPO, "gpurun_out")
MEMPLAN = os.path.join(REPO, "build", "memplan")
SCRATCH = "/tmp/ptk_runtime_bench"

BASE = {"h2d_bw": 5.5e10, "d2h_bw": 5.5e10, "coll_alpha": 2e-5, "coll_bw": 7.7e11,
        "world_size": 1, "gpu_mem": 180_000_000_000, "cpu_mem": 1_000_000_000_000,
        "cpu_optim_rate": 1e9, "gpu_optim_rate": 1e11}

# (name, gen-trace args, forced config or None for the planner's choice)
CASES = [
    ("gpt2-1.5b_b8 all-persistent (cfg2)", ["--spec", "golden:gpt2_1.5b_spec.json", "--batch", "8"],
     {"n_persist": "all", "n_buffer": 0}),
    ("gpt2-10b shape, 8 blocks, b8: np=0 nb=3 (cfg3 slice: 402 MB block chunks offloaded)",
     ["--spec", "spec:gpt2-10b-8blk", "--batch", "8"], {"n_persist": 0, "n_buffer": 3}),
    ("gpt2-10b shape, 8 blocks, b8: planner's choice under the measured profile",
     ["--spec", "spec:gpt2-10b-8blk", "--batch", "8"], None),
    ("gpt2-1b b2 (cfg1): np=1 nb=2 (reference Gantt case)", ["--model", "gpt2-1b", "--batch", "2"],
     {"n_persist": 1, "n_buffer": 2}),
]


def run(args, **kw):
    return subprocess.run([MEMPLAN] + args, check=True, capture_output=True, text=True, **kw).stdout


def main():
    from paper_2406_08334_b200 import runtime
    os.makedirs(SCRATCH, exist_ok=True)
    os.makedirs(OUT, exist_ok=True)
    base = os.path.join(SCRATCH, "base.json")
    json.dump(BASE, open(base, "w"))
    measured_path = os.path.join(OUT, "b200x1_measured.json")
    hw = runtime.measure_profile(base, measured_path)
    print("measured profile:", json.dumps(hw), flush=True)
    spec10 = os.path.join(SCRATCH, "gpt2-10b-8blk.json")
    json.dump({"hidden_size": 4096, "n_blocks": 8, "n_heads": 32}, open(spec10, "w"))
    lines = []
    for name, targs, forced in CASES:
        targs = [a.replace("golden:", os.path.join(REPO, "tests", "golden") + "/")
                  .replace("spec:gpt2-10b-8blk", spec10) for a in targs]
        trace = os.path.join(SCRATCH, "trace.json")
        run(["gen-trace"] + targs + ["-o", trace])
        layout = json.loads(run(["pack", "--trace", trace]))
        plan = os.path.join(SCRATCH, "plan.json")
        if forced is None:
            out = json.loads(run(["plan", "--trace", trace, "--hw", measured_path]))
            cfg = out["config"]
        else:
            n = layout["n_chunk"]
            np_ = n if forced["n_persist"] == "all" else forced["n_persist"]
            tr = json.load(open(trace))
            # n_interval only matters with swap blocks (none in the forced cases)
            cfg = {"s_chunk": layout["s_chunk"], "n_chunk": n, "n_persist": np_,
                   "n_buffer": forced["n_buffer"], "n_block": tr["n_blocks"], "n_interval": 1,
                   "n_swap": 0, "n_checkpoint": 0}
        json.dump(cfg, open(plan, "w"))
        res = runtime.execute_plan(trace, plan, measured_path, compute_scale=1.0, iterations=3)
        meta = json.load(open(trace))["meta"]
        tokens = int(meta["batch_size"]) * int(meta["seq_len"])
        row = {"case": name, "config": cfg, "measured_t_iter": res["t_iter"],
               "estimate_t_iter": res["estimate_t_iter"],
               "rel_err": abs(res["t_iter"] - res["estimate_t_iter"]) / res["estimate_t_iter"],
               "tokens_per_s_standin_compute": tokens / res["t_iter"],
               "h2d_GB": res["h2d_bytes"] / 1e9, "d2h_GB": res["d2h_bytes"] / 1e9,
               "gpu_optim_ms": res["gpu_optim_ns"] / 1e6, "cpu_optim_ms": res["cpu_optim_ns"] / 1e6,
               "device_GB": res["device_bytes"] / 1e9, "pinned_host_GB": res["pinned_host_bytes"] / 1e9,
               "measured_m_peak": res["m_peak"], "estimate_m_peak": res["estimate_m_peak"],
               "events": len(res["timeline"])}
        print(json.dumps(row), flush=True)
        lines.append(row)
        with open(os.path.join(OUT, f"runtime_timeline_{len(lines)}.csv"), "w") as f:
            f.write(res["timeline_csv"])
    with open(os.path.join(OUT, "runtime_bench.jsonl"), "w") as f:
        for row in lines:
            f.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
