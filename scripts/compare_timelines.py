#!/usr/bin/env python3
"""Measured training timeline vs the simulator's timeline of the same plan.

    python scripts/compare_timelines.py REAL.csv SIM.csv [--blocks-per-row 8]

REAL = `train_large.py --timeline` output (per-block compute events);
SIM = `memplan simulate --timeline-csv` (per-operator compute events: op i of
a synthesized trace belongs to block (i-1)//8, op 0 is the embedding). Prints
per-block forward / backward intervals and per-chunk upload / offload / host
update intervals side by side (ms from each timeline's origin), and where the
real iteration falls behind the simulated one.
"""
from __future__ import annotations

import argparse
import os
import re
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def intervals(rows, per_op: bool):
    """{(kind, key): (start_ns, end_ns)} with key = block (compute) or chunk."""
    out: dict = {}
    opened: dict = {}
    for ns, resource, event, subject in rows:
        m = re.match(r"(\w+)_(start|end)$", event)
        if not m:
            continue
        kind, edge = m.groups()
        if kind in ("fwd", "bwd", "recompute"):
            if per_op:
                mo = re.search(r"op=(\d+)", subject)
                if mo is None:
                    mb = re.search(r"block=(\d+)", subject)
                    if mb is None:
                        continue
                    key = int(mb.group(1))
                else:
                    i = int(mo.group(1))
                    key = (i - 1) // 8 if i >= 1 else -1
            else:
                mb = re.search(r"block=(\d+)", subject)
                if mb is None:
                    continue
                key = int(mb.group(1))
            if kind == "recompute":
                kind = "bwd"
        else:
            mc = re.search(r"chunk=(\d+)", subject)
            if mc is None:
                continue
            key = int(mc.group(1))
            if subject.endswith(" prev"):
                kind += "(prev)"
        k = (kind, key)
        if edge == "start":
            if k not in out:
                out[k] = [ns, ns]
            else:
                out[k][0] = min(out[k][0], ns)
            opened[k] = ns
        else:
            if k not in out:
                out[k] = [ns, ns]
            out[k][1] = max(out[k][1], ns)
    return {k: tuple(v) for k, v in out.items()}


def main():
    from paper_2406_08334_b200.timeline import last_iteration, read_csv
    ap = argparse.ArgumentParser()
    ap.add_argument("real")
    ap.add_argument("sim")
    args = ap.parse_args()
    real, sim = read_csv(args.real), read_csv(args.sim)
    starts = [ns for ns, _, e, _ in real if e == "iter_start"]
    if starts:   # several recorded iterations: compare the last (steady state)
        print(f"{len(starts)} recorded iterations, comparing the last "
              f"(starts at {max(starts) / 1e6:.1f} ms); 'prev' = carried over from the one before")
    real = last_iteration(real)
    r, s = intervals(real, per_op=False), intervals(sim, per_op=True)
    ms = lambda ns: ns / 1e6  # noqa: E731
    print(f"iteration end: real {ms(max(t for t, *_ in real)):.1f} ms, "
          f"simulated {ms(max(t for t, *_ in sim)):.1f} ms")
    blocks = sorted({k for kind, k in r if kind in ("fwd", "bwd") and k >= 0})
    print("\nblock | real fwd (ms)      | sim fwd            | real bwd            | sim bwd")
    for b in blocks:
        cells = []
        for kind in ("fwd", "bwd"):
            for src in (r, s):
                iv = src.get((kind, b))
                cells.append(f"{ms(iv[0]):8.1f}-{ms(iv[1]):8.1f}" if iv else " " * 17)
        print(f"{b:5d} | " + " | ".join(cells))
    chunks = sorted({k for kind, k in list(r) + list(s) if kind in ("upload", "offload", "update",
                                                                     "optim", "update(prev)")})
    print("\nchunk | kind    | real (ms)           | simulated")
    for c in chunks:
        for kind in ("update(prev)", "upload", "offload", "update", "optim"):
            a, b = r.get((kind, c)), s.get((kind, c))
            if a is None and b is None:
                continue
            fa = f"{ms(a[0]):8.1f}-{ms(a[1]):8.1f}" if a else " " * 17
            fb = f"{ms(b[0]):8.1f}-{ms(b[1]):8.1f}" if b else " " * 17
            print(f"{c:5d} | {kind:7s} | {fa} | {fb}")


if __name__ == "__main__":
    main()
