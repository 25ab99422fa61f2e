#!/usr/bin/env python3
"""HBM efficiency of the fused RS -> Adam -> AG peer kernel on ONE GPU.

W virtual ranks live on one device (each its own ChunkSet: full bf16 param +
grad chunk buffers, fp32 master/m/v of its shard) and the kernel of rank r
reads the owned shard of every rank's gradient chunk and stores its bf16
result into every rank's parameter chunk -- exactly the memory operations it
performs over NVLink on a real W-GPU node, here all on local HBM. One "step"
= the W launches (one per virtual rank) over every chunk.

Algorithmic bytes per owned element: master/m/v read + write (24 B), W grad
reads (2W B), W param writes (2W B); summed over ranks: P * (24 + 4W) bytes.
This measures how close the kernel's structure (128-bit vector loads of W
peers, fp32 rank-order sum, push all-gather) comes to the HBM roofline when
nothing but HBM bounds it; over NVLink the (W-1)/W remote share is bounded by
the links instead.

    python scripts/fused_virtual_bench.py --chunk-mib 512 --worlds 1,2,4,8
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunk-mib", type=int, default=512)
    ap.add_argument("--chunks", type=int, default=1,
                    help="chunks per step (one table launch per virtual rank walks all of them)")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    peak = float(peaks["hbm_gbs"])
    dev = torch.device("cuda", 0)
    p = args.chunk_mib * (1 << 20) // 2
    rows = []
    for w in map(int, args.worlds.split(",")):
        sets = [ChunkSet([p] * args.chunks, world=w, rank=r, device=dev, mode="fused") for r in range(w)]
        for cs in sets:
            cs.init_synthetic()
            cs.fill_grads(0)
            cs.attach_virtual_peers(sets)
        hyper = AdamHyper(lr=1e-3)
        for _ in range(args.warmup):
            for cs in sets:
                cs.step(hyper, with_stats=False)
        torch.cuda.synchronize()
        launches0 = nat.launch_count()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(args.steps):
                for cs in sets:
                    cs.step(hyper, with_stats=False)
        launches = nat.launch_count() - launches0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        alg = p * args.chunks * (24 + 4 * w)
        gbs = alg / (ms * 1e-3) / 1e9
        row = {"kernel": nat.raw.ptk_fused_kernel_name().decode() + f" W={w}",
               "virtual_ranks": w, "chunk_params": p, "chunks": args.chunks,
               "ms_per_step": round(ms, 4), "algorithmic_bytes_per_step": alg,
               "achieved_gbs": round(gbs, 1), "peak_gbs": peak, "frac": round(gbs / peak, 4),
               "launches_per_step": launches // args.steps,
               "timing": "CUDA graph of the steps, one replay"}
        print(json.dumps(row), flush=True)
        rows.append(row)
        del g, sets
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", "fused_virtual.jsonl"), "a") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
