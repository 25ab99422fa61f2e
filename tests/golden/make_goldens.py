"""Generate the golden fixtures of the planner from the REFERENCE itself.

Runs oracle/_ref/memplan — the unmodified reference CLI built from
/root/reference/proj by oracle/Makefile — on the BASELINE configs and on the
reference's own standard fixtures, and writes its byte-exact outputs here.
Only run in the build container (the GPU box has no /root/reference; the
committed outputs travel instead):

    make -C oracle ref && python tests/golden/make_goldens.py

Cases:
  cfg1  gpt2-1b b2            reference test model (test_cost.cpp:260-262)
  cfg2  GPT-2 1.5B b8         {hidden 1600, L48, 25 heads}; all persistent
  cfg3  gpt2-10b b8           np=0 nb=3, w=2/4/8
  cfg4  llama-13b b8          cost-model-chosen plan, B200-like profile
plus the paper testbeds (rtx3090x4 / a100x4 / a100x1) for search winners.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(REPO, "oracle", "_ref", "memplan")
TMP = "/tmp/ptk_goldens"

# B200-like flag overrides: not measured values.
B200_LIKE = ["--gpu-mem", "180000000000", "--coll-bw", "9e11", "--h2d-bw", "5.5e10",
             "--d2h-bw", "5.5e10", "--cpu-mem", "2000000000000"]

TRACES = {
    "gpt2-1b_b2": ["--model", "gpt2-1b", "--batch", "2"],
    "gpt2-1.5b_b8": ["--spec", os.path.join(HERE, "gpt2_1.5b_spec.json"), "--batch", "8"],
    "gpt2-10b_b8": ["--model", "gpt2-10b", "--batch", "8"],
    "llama-13b_b8": ["--model", "llama-13b", "--batch", "8"],
    "gpt2-10b_b6": ["--model", "gpt2-10b", "--batch", "6"],
}

# (name, verb, trace, args)
CASES = [
    ("pack_gpt2-1b_b2", "pack", "gpt2-1b_b2", []),
    ("pack_gpt2-1.5b_b8", "pack", "gpt2-1.5b_b8", []),
    ("pack_gpt2-10b_b8", "pack", "gpt2-10b_b8", []),
    ("pack_llama-13b_b8", "pack", "llama-13b_b8", []),
    ("pack_gpt2-10b_b8_grid", "pack", "gpt2-10b_b8", ["--grid", "512Mi,1Gi,2Gi"]),
    ("plan_gpt2-1b_b2_a100x1", "plan", "gpt2-1b_b2", ["--hw", "a100x1"]),
    ("plan_gpt2-1b_b2_a100x4", "plan", "gpt2-1b_b2", ["--hw", "a100x4"]),
    ("plan_gpt2-1b_b2_rtx3090x4", "plan", "gpt2-1b_b2", ["--hw", "rtx3090x4"]),
    ("plan_gpt2-10b_b8_rtx3090x4", "plan", "gpt2-10b_b8", ["--hw", "rtx3090x4"]),
    ("plan_gpt2-10b_b8_a100x4", "plan", "gpt2-10b_b8", ["--hw", "a100x4"]),
    ("plan_gpt2-1.5b_b8_b200x1", "plan", "gpt2-1.5b_b8",
     ["--hw", "a100x1"] + B200_LIKE + ["--gpu-optim-rate", "2e11", "--world-size", "1"]),
    ("plan_gpt2-1.5b_b8_b200x8", "plan", "gpt2-1.5b_b8",
     ["--hw", "a100x1"] + B200_LIKE + ["--gpu-optim-rate", "2e11", "--world-size", "8"]),
    ("plan_gpt2-10b_b8_b200x8", "plan", "gpt2-10b_b8",
     ["--hw", "a100x4"] + B200_LIKE + ["--world-size", "8"]),
    ("plan_gpt2-10b_b8_b200x2_gpu2e11", "plan", "gpt2-10b_b8",
     ["--hw", "a100x4"] + B200_LIKE + ["--gpu-optim-rate", "2e11", "--world-size", "2"]),
    ("plan_llama-13b_b8_b200x8", "plan", "llama-13b_b8",
     ["--hw", "a100x4"] + B200_LIKE + ["--gpu-optim-rate", "2e11", "--world-size", "8"]),
    ("estimate_gpt2-1.5b_b8_allpersist_w1", "estimate", "gpt2-1.5b_b8",
     ["--hw", "a100x1"] + B200_LIKE + ["--gpu-optim-rate", "2e11", "--world-size", "1",
                                       "--n-persist", "3"]),
    ("estimate_gpt2-1.5b_b8_allpersist_w8", "estimate", "gpt2-1.5b_b8",
     ["--hw", "a100x1"] + B200_LIKE + ["--gpu-optim-rate", "2e11", "--world-size", "8",
                                       "--n-persist", "3"]),
    ("simulate_gpt2-1.5b_b8_allpersist_w8", "simulate", "gpt2-1.5b_b8",
     ["--hw", "a100x1"] + B200_LIKE + ["--gpu-optim-rate", "2e11", "--world-size", "8",
                                       "--n-persist", "3"]),
    ("estimate_gpt2-10b_b8_np0nb3_w2", "estimate", "gpt2-10b_b8",
     ["--hw", "a100x4"] + B200_LIKE + ["--world-size", "2", "--n-persist", "0", "--n-buffer", "3"]),
    ("estimate_gpt2-10b_b8_np0nb3_w8", "estimate", "gpt2-10b_b8",
     ["--hw", "a100x4"] + B200_LIKE + ["--world-size", "8", "--n-persist", "0", "--n-buffer", "3"]),
    ("simulate_gpt2-10b_b8_np0nb3_w8", "simulate", "gpt2-10b_b8",
     ["--hw", "a100x4"] + B200_LIKE + ["--world-size", "8", "--n-persist", "0", "--n-buffer", "3"]),
    ("simulate_gpt2-1b_b2_np1nb2_a100x4", "simulate", "gpt2-1b_b2",
     ["--hw", "a100x4", "--n-persist", "1", "--n-buffer", "2"]),
    ("simulate_gpt2-1b_b2_np1nb2_ns1nc20_rtx3090x4", "simulate", "gpt2-1b_b2",
     ["--hw", "rtx3090x4", "--n-persist", "1", "--n-buffer", "2", "--n-swap", "1",
      "--n-checkpoint", "20"]),
    ("validate_gpt2-10b_b6_rtx3090x4", "validate", "gpt2-10b_b6",
     ["--hw", "rtx3090x4", "--samples", "12", "--seed", "0"]),
    ("sweep_gpt2-1b_b2_a100x4", "sweep", "gpt2-1b_b2",
     ["--hw", "a100x4", "--n-persist", "0:4", "--n-buffer", "-1:-1", "--n-checkpoint", "0:8"]),
]

# simulate cases also record the event timeline CSV
TIMELINES = {"simulate_gpt2-1b_b2_np1nb2_a100x4", "simulate_gpt2-10b_b8_np0nb3_w8",
             "simulate_gpt2-1b_b2_np1nb2_ns1nc20_rtx3090x4"}


def run(args, **kw):
    return subprocess.run([REF] + args, check=True, capture_output=True, text=True, **kw)


def main() -> int:
    if not os.path.exists(REF):
        print(f"missing {REF}; run `make -C oracle ref` first", file=sys.stderr)
        return 1
    os.makedirs(TMP, exist_ok=True)
    traces = {}
    for name, args in TRACES.items():
        path = os.path.join(TMP, f"trace_{name}.json")
        run(["gen-trace"] + args + ["-o", path])
        traces[name] = path
    manifest = {"generator": "oracle/_ref/memplan (reference, unmodified)", "traces": TRACES,
                "cases": []}
    for name, verb, trace, args in CASES:
        extra = []
        if name in TIMELINES:
            extra = ["--timeline-csv", os.path.join(HERE, f"{name}.timeline.csv")]
        out = run([verb, "--trace", traces[trace]] + args + extra)
        ext = "csv" if verb in ("validate", "sweep") else "json"
        with open(os.path.join(HERE, f"{name}.{ext}"), "w") as f:
            f.write(out.stdout)
        manifest["cases"].append({"name": name, "verb": verb, "trace": trace, "args": args,
                                  "output": f"{name}.{ext}",
                                  "timeline": f"{name}.timeline.csv" if extra else None})
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
        f.write("\n")
    print(f"wrote {len(CASES)} golden outputs to {HERE}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
