#!/usr/bin/env python3
"""Soak run of the chunked training step: N iterations of the cfg2 model
(GPT-2 1.5B b8, all chunks persistent, CUDA-graph forward/backward) on a
learnable synthetic stream (next token = token + 1), recording the loss
every 25 iterations and the device memory in use, so a leak or a diverging
update shows up. One JSON line.

    python scripts/train_soak.py --iters 300
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--workload", default="gpt2-1.5b_b8")
    args = ap.parse_args()
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, GraphedTrainStep
    dev = torch.device("cuda", 0)
    trace, layout = planner.trace_for(args.workload), planner.layout_for(args.workload)
    cs = ChunkSet([c["used_bytes"] // 2 for c in layout["chunks"]], device=dev)
    shape = GPT2Shape.from_trace(trace)
    model = ChunkedGPT2(shape, layout, cs, trace["ops"])
    model.init_weights(0)
    batch = int(trace["meta"]["batch_size"])
    g = torch.Generator(device=dev).manual_seed(0)
    hyper = AdamHyper(lr=3e-4, weight_decay=0.01, adamw=True)

    def batch_xy():
        x = torch.randint(0, shape.vocab, (batch, shape.seq), device=dev, generator=g)
        return x, (x + 1) % shape.vocab

    x, y = batch_xy()
    step = GraphedTrainStep(model, x, y)
    losses, mem = [], []
    t0 = time.perf_counter()
    for i in range(args.iters):
        x, y = batch_xy()
        loss = step(x, y, hyper)
        if i % 25 == 0 or i == args.iters - 1:
            losses.append((i, round(float(loss), 4)))
            mem.append((i, round(torch.cuda.memory_allocated() / 1e9, 3)))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    sumsq, bad = cs.grad_stats()
    print(json.dumps({"workload": args.workload, "iters": args.iters,
                      "tokens_per_s_wall": round(args.iters * batch * shape.seq / wall, 1),
                      "loss": losses, "allocated_GB": mem,
                      "last_grad_norm": round(sumsq ** 0.5, 4), "nonfinite": bad}))


if __name__ == "__main__":
    main()
