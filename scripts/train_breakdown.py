#!/usr/bin/env python3
"""Where a chunked training iteration spends its device time: torch.profiler
(CUPTI kernel records) over 3 host-launched iterations of the cfg1 / cfg2
model, kernels grouped into GEMM, attention, chunk step (libptk), gradient
stash copies, elementwise/norm and the rest.

    python scripts/train_breakdown.py --workload cfg2
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
MODELS = {"cfg2": "gpt2-1.5b_b8", "cfg1": "gpt2-1b_b2"}


def category(name: str) -> str:
    n = name.lower()
    if "ptk::" in n or "chunk_adam" in n or "stats_reset" in n:
        return "chunk step (libptk)"
    if "gemm" in n or "cutlass" in n or "nvjet" in n or "sm100" in n and "xmma" in n or "cublas" in n:
        return "GEMM (cuBLAS)"
    if "cudnn" in n or "flash" in n or "fmha" in n or "attention" in n or "sdpa" in n:
        return "attention"
    if "copy" in n or "memcpy" in n:
        return "copies (grad stash etc.)"
    if "norm" in n or "elementwise" in n or "reduce" in n or "softmax" in n or "cross_entropy" in n \
            or "nll" in n or "gelu" in n or "embedding" in n or "cat" in n:
        return "elementwise / norm / loss"
    return "other"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2", choices=sorted(MODELS))
    args = ap.parse_args()
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step
    dev = torch.device("cuda", 0)
    name = MODELS[args.workload]
    trace, layout = planner.trace_for(name), planner.layout_for(name)
    cs = ChunkSet([c["used_bytes"] // 2 for c in layout["chunks"]], device=dev)
    shape = GPT2Shape.from_trace(trace)
    model = ChunkedGPT2(shape, layout, cs, trace["ops"])
    model.init_weights(0)
    batch = int(trace["meta"]["batch_size"])
    x = torch.randint(0, shape.vocab, (batch, shape.seq), device=dev)
    y = (x + 1) % shape.vocab
    hyper = AdamHyper(lr=1e-4)
    for _ in range(3):
        train_step(model, x, y, hyper)
    torch.cuda.synchronize()
    iters = 3
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(iters):
            train_step(model, x, y, hyper)
        torch.cuda.synchronize()
    agg: dict = collections.defaultdict(float)
    top: dict = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            t = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
            agg[category(ev.name)] += t / 1e3 / iters
            top[ev.name[:90]] += t / 1e3 / iters
    total = sum(agg.values())
    out = {"workload": args.workload, "model": name, "device_ms_per_iter": round(total, 2),
           "by_category_ms": {k: round(v, 2) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])},
           "top_kernels_ms": {k: round(v, 2) for k, v in sorted(top.items(), key=lambda kv: -kv[1])[:12]}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
