#!/usr/bin/env python3
"""Search / simulate wall time: this build's `memplan` vs the reference's own
binary (oracle/_ref/memplan, compiled from /root/reference by oracle/Makefile),
same inputs, outputs compared byte for byte.

Runs on the host only (no GPU). Writes one JSON line per case to stdout.
  python scripts/planner_bench.py [--reps 3] [--threads N ...]
"""
import argparse
import json
import os
import subprocess
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = os.path.join(REPO, "build", "memplan")
REF = os.path.join(REPO, "oracle", "_ref", "memplan")
B200 = ["--hw", "a100x4", "--gpu-mem", "180000000000", "--coll-bw", "9e11", "--h2d-bw", "5.5e10",
        "--d2h-bw", "5.5e10", "--cpu-mem", "2000000000000"]
CASES = [
    # (name, trace args, verb args)
    ("cfg3 gpt2-10b b8 plan, B200-like w=8", ["--model", "gpt2-10b", "--batch", "8"],
     ["plan"] + B200 + ["--gpu-optim-rate", "2e11", "--world-size", "8"]),
    ("cfg3 gpt2-10b b8 plan, rtx3090x4", ["--model", "gpt2-10b", "--batch", "8"],
     ["plan", "--hw", "rtx3090x4"]),
    ("cfg4 llama-13b b8 plan, B200-like", ["--model", "llama-13b", "--batch", "8"],
     ["plan"] + B200),
    ("gpt2-10b b8 validate 50 (estimate + simulate each), a100x4",
     ["--model", "gpt2-10b", "--batch", "8"],
     ["validate", "--hw", "a100x4", "--samples", "50"]),
]


def timed(cmd, reps, env=None):
    best, out = 1e30, None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = subprocess.run(cmd, capture_output=True, text=True, env=env)
        dt = time.perf_counter() - t0
        if r.returncode != 0:
            raise RuntimeError(f"{cmd[0]} failed: {r.stderr}")
        best, out = min(best, dt), r.stdout
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--threads", type=int, nargs="*", default=[1, os.cpu_count()])
    args = ap.parse_args()
    if not (os.path.exists(OURS) and os.path.exists(REF)):
        raise SystemExit("build first: make planner && make -C oracle ref")
    tmp = os.path.join(REPO, "build", "planner_bench")
    os.makedirs(tmp, exist_ok=True)
    for name, targs, vargs in CASES:
        trace = os.path.join(tmp, "trace_" + "_".join(targs[1::2]) + ".json")
        subprocess.run([OURS, "gen-trace"] + targs + ["-o", trace], check=True)
        cmd_tail = [vargs[0], "--trace", trace] + vargs[1:]
        t_ref, out_ref = timed([REF] + cmd_tail, args.reps)
        row = {"case": name, "reference_s": round(t_ref, 3)}
        for th in args.threads:
            env = dict(os.environ, MEMPLAN_THREADS=str(th))
            t, out = timed([OURS] + cmd_tail, args.reps, env)
            row[f"ours_{th}t_s"] = round(t, 3)
            row[f"speedup_{th}t"] = round(t_ref / t, 2)
            row[f"identical_{th}t"] = out == out_ref
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
