#!/usr/bin/env python3
"""Plain-PyTorch baseline for the chunked training step: the same model (the
trace's operators, train.block_forward / head_loss) with ordinary bf16 leaf
parameters, fp32 master copies and torch.optim.AdamW(fused=True) -- the
standard mixed-precision recipe -- timed like bench.py's `train`.

    python scripts/train_torch_baseline.py --workload cfg2 --steps 10 --warmup 3

Per iteration: forward + backward (identical kernels to the chunked model),
grads cast to fp32 as the masters' grads, fused AdamW over the fp32 masters,
masters copied back to the bf16 parameters (torch._foreach_copy_). Prints one JSON
line (tokens/s, ms/iter) to set beside bench.py's train block.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import types

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

MODELS = {"cfg2": "gpt2-1.5b_b8", "cfg1": "gpt2-1b_b2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2", choices=sorted(MODELS))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, op_param_shapes
    dev = torch.device("cuda", 0)
    trace = planner.trace_for(MODELS[args.workload])
    shape = GPT2Shape.from_trace(trace)
    g = torch.Generator(device=dev).manual_seed(0)
    params: dict[str, torch.Tensor] = {}
    blocks = [dict() for _ in range(shape.blocks)]
    for name, plist in op_param_shapes(shape):
        where = int(name.split(".")[1]) if "." in name else None
        for pname, pshape in plist:
            t = torch.empty(pshape, dtype=torch.bfloat16, device=dev)
            if pname.endswith("_w") and len(pshape) == 2 or pname in ("wte", "wpe", "head_w"):
                t.normal_(0.0, 0.02, generator=g)
            elif pname in ("ln1_w", "ln2_w"):
                t.fill_(1.0)
            else:
                t.zero_()
            t.requires_grad_(True)
            (params if where is None else blocks[where])[pname] = t
    model = types.SimpleNamespace(shape=shape, params=params, blocks=blocks)
    leaves = list(params.values()) + [p for b in blocks for p in b.values()]
    masters = [p.detach().float().clone() for p in leaves]
    opt = torch.optim.AdamW(masters, lr=1e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01,
                            fused=True)
    batch = int(trace["meta"]["batch_size"])
    n_iter = args.warmup + args.steps
    tokens = torch.randint(0, shape.vocab, (n_iter, batch, shape.seq), device=dev, generator=g)
    targets = (tokens + 1) % shape.vocab

    def step(i):
        loss = ChunkedGPT2.loss(model, tokens[i], targets[i])
        loss.backward()
        grads = [p.grad for p in leaves]
        for m, gr in zip(masters, grads):
            m.grad = gr.float()
        opt.step()
        with torch.no_grad():
            torch._foreach_copy_(leaves, masters)
        for p in leaves:
            p.grad = None
        for m in masters:
            m.grad = None
        return loss.detach()

    losses = [step(i) for i in range(args.warmup)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.warmup, n_iter):
        losses.append(step(i))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(json.dumps({"baseline": "plain PyTorch: bf16 params, fp32 masters, "
                                  "torch.optim.AdamW(fused=True)",
                      "model": MODELS[args.workload], "tokens_per_s": round(batch * shape.seq / (ms * 1e-3), 1),
                      "ms_per_iter": round(ms, 3), "iters": args.steps,
                      "loss_first": round(float(losses[0]), 4),
                      "loss_last": round(float(losses[-1]), 4),
                      "peak_allocated_GB": round(torch.cuda.max_memory_allocated() / 1e9, 2)}))


if __name__ == "__main__":
    main()
