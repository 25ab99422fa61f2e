#!/usr/bin/env python3
"""Host Adam (K6, ptk_cpu_adam) rate vs OpenMP thread count on this host,
over pinned shards as the ChunkPool uses them, alone and with a concurrent
pinned H2D + D2H copy stream (the DMA traffic of an offloaded iteration).

    python scripts/host_adam_threads.py --params 268435456
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import threading
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--params", type=int, default=256 * 1024 * 1024)
    ap.add_argument("--threads", default="4,8,12,14,15,16")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import vp
    n = args.params
    pin = dict(pin_memory=True)
    master = torch.randn(n, **pin) * 0.05
    m = torch.zeros(n, **pin)
    v = torch.zeros(n, **pin)
    g = (torch.randn(n) * 1e-3).to(torch.bfloat16).pin_memory()
    p = torch.empty(n, dtype=torch.bfloat16, **pin)
    cfg = nat.adam_config(lr=1e-3, step=1)

    # concurrent DMA: 1 GiB pinned <-> device, both directions, on two streams
    dev = torch.device("cuda", 0)
    hb = torch.empty(1 << 29, dtype=torch.bfloat16, **pin)
    db = torch.empty(1 << 29, dtype=torch.bfloat16, device=dev)
    hb2 = torch.empty_like(hb, **pin)
    stop = threading.Event()

    def dma():
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        while not stop.is_set():
            with torch.cuda.stream(s1):
                db.copy_(hb, non_blocking=True)
            with torch.cuda.stream(s2):
                hb2.copy_(db, non_blocking=True)
            s1.synchronize()
            s2.synchronize()

    def rate(threads):
        best = 0.0
        for _ in range(args.reps):
            t0 = time.perf_counter()
            nat.raw.ptk_cpu_adam(ctypes.byref(cfg), vp(master), vp(m), vp(v), vp(g), vp(p), n,
                                 threads, None, None)
            best = max(best, n / (time.perf_counter() - t0))
        return best

    rows = []
    for t in map(int, args.threads.split(",")):
        alone = rate(t)
        stop.clear()
        th = threading.Thread(target=dma)
        th.start()
        time.sleep(0.2)
        busy = rate(t)
        stop.set()
        th.join()
        row = {"threads": t, "params_per_s_alone": round(alone / 1e9, 3),
               "params_per_s_with_dma": round(busy / 1e9, 3),
               "host_GBs_alone_28B": round(28 * alone / 1e9, 1), "cpus": os.cpu_count()}
        print(json.dumps(row), flush=True)
        rows.append(row)


if __name__ == "__main__":
    main()
