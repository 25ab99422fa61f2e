#!/usr/bin/env python3
"""HBM efficiency of the non-persistent chunks' peer exchange on ONE GPU with
W virtual ranks (every "peer" buffer on this device): ptk_peer_reduce_scatter_f32
(per rank: W bf16 shard reads + one fp32 shard write = (2W + 4) B per owned
element) and ptk_peer_allgather (copy-engine pulls of W-1 shards = 2 x 2 B per
pulled element, read + write). On a W-GPU node the (W-1)/W remote share of
both crosses NVLink instead (770 GB/s per direction).

    python scripts/peer_exchange_bench.py --chunk-mib 512 --worlds 2,4,8
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import vp
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunk-mib", type=int, default=512)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda", 0)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    n = args.chunk_mib << 19  # bf16 elements per chunk
    for w in map(int, args.worlds.split(",")):
        shard = nat.shard_elems(n, w)
        bufs = [torch.zeros(shard * w, dtype=torch.int16, device=dev) for _ in range(w)]
        ptrs = (ctypes.c_void_p * nat.PTK_MAX_PEERS)(*[b.data_ptr() for b in bufs])
        out = torch.empty(shard, dtype=torch.float32, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def timed(fn):
            fn()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.reps

        def rs():   # every rank's reduce, one after the other (a W-GPU step)
            for r in range(w):
                nat.lib.ptk_peer_reduce_scatter_f32(ptrs, w, r, shard, vp(out), s)

        def ag():
            for r in range(w):
                nat.lib.ptk_peer_allgather(ptrs, w, r, 2 * shard, s)

        ms_rs, ms_ag = timed(rs), timed(ag)
        b_rs = w * shard * (2 * w + 4)
        b_ag = w * (w - 1) * shard * 2 * 2
        for name, ms, b in (("peer_reduce_scatter_f32", ms_rs, b_rs), ("peer_allgather", ms_ag, b_ag)):
            gbs = b / (ms * 1e-3) / 1e9
            print(json.dumps({"op": name, "virtual_ranks": w, "chunk_mib": args.chunk_mib,
                              "ms_per_step": round(ms, 4), "algorithmic_bytes": b,
                              "achieved_gbs": round(gbs, 1), "frac_of_measured_hbm": round(gbs / peak, 4)}))
        del bufs, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
