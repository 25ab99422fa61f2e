"""Measured timeline of a training iteration in the simulator's event schema.

`memplan simulate --timeline-csv` writes one row per modeled event:
`time_ns,resource,event,subject` (proj/src/sim.cpp:187-189,765-797 — gpu
fwd/bwd per operator, h2d upload / d2h offload / cpu update / gpu optim per
chunk, swap chains). `Timeline` records the same events from a REAL training
iteration of the chunked model: device events as CUDA events on the stream
that carries the work (so their times are when the device reached them), host
events (the host Adam of offloaded chunks) with the host clock, both relative
to one origin taken right after a device synchronisation. Compute is recorded
per block (`subject` "block=b") rather than per operator; chunk subjects are
1-based like the simulator's ("chunk=c").

Disabled (the default: `model.timeline = None`) it costs nothing.
"""
from __future__ import annotations

import csv
import json
import threading
import time

import torch


class Timeline:
    def __init__(self):
        self._rows: list = []
        self._lock = threading.Lock()
        self._origin = None
        self._t0 = 0.0

    def begin(self) -> None:
        """Start an iteration's record (synchronises the device once)."""
        torch.cuda.synchronize()
        self._rows = []
        self._origin = torch.cuda.Event(enable_timing=True)
        self._origin.record()
        torch.cuda.synchronize()
        self._t0 = time.perf_counter()

    def gpu(self, stream, resource: str, event: str, subject: str) -> None:
        """An event at the point `stream` reaches now (device time)."""
        if self._origin is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream if stream is not None else torch.cuda.current_stream())
        with self._lock:
            self._rows.append((e, resource, event, subject))

    def host(self, resource: str, event: str, subject: str) -> None:
        """An event at this moment of the host clock (e.g. host Adam)."""
        if self._origin is None:
            return
        t = time.perf_counter()
        with self._lock:
            self._rows.append((t, resource, event, subject))

    def end(self) -> list[tuple[int, str, str, str]]:
        """Finish the record: rows (time_ns, resource, event, subject), sorted."""
        torch.cuda.synchronize()
        out = []
        with self._lock:
            rows, self._rows = self._rows, []
        for when, resource, event, subject in rows:
            if isinstance(when, float):
                ns = int(round((when - self._t0) * 1e9))
            else:
                ns = int(round(self._origin.elapsed_time(when) * 1e6))
            out.append((ns, resource, event, subject))
        self._origin = None
        out.sort(key=lambda r: r[0])
        return out


def write_csv(rows, path: str) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f, quoting=csv.QUOTE_MINIMAL)
        w.writerow(["time_ns", "resource", "event", "subject"])
        for ns, resource, event, subject in rows:
            w.writerow([ns, resource, event, subject])


def write_chrome_trace(rows, path: str) -> None:
    """The measured timeline as Chrome-trace instant events, in the exact
    layout `memplan simulate --timeline` writes for a simulated one
    (proj/src/sim.cpp:765-797): one thread row per resource in order of
    first use, ts in microseconds, name "<event> <subject>" -- so a measured
    and a simulated iteration open side by side in chrome://tracing."""
    rows_of: dict[str, int] = {}
    events = []
    for ns, resource, event, subject in rows:
        tid = rows_of.setdefault(resource, len(rows_of) + 1)
        events.append({"name": f"{event} {subject}", "ph": "i", "pid": 1, "s": "t",
                       "tid": tid, "ts": ns / 1000.0})
    with open(path, "w") as f:
        json.dump(events, f, indent=1)
        f.write("\n")


def read_csv(path: str) -> list[tuple[int, str, str, str]]:
    with open(path) as f:
        return [(int(r["time_ns"]), r["resource"], r["event"], r["subject"])
                for r in csv.DictReader(f)]


def last_iteration(rows) -> list[tuple[int, str, str, str]]:
    """The rows of the last recorded iteration (from its `iter_start` event),
    re-based to start at 0. Intervals still open from the previous iteration
    (e.g. its host Adam) are kept from 0 with " prev" appended to the subject."""
    starts = [ns for ns, _, e, _ in rows if e == "iter_start"]
    if not starts:
        return [r for r in rows if r[2] != "iter_start"]
    last = max(starts)
    opened = set()
    for ns, resource, event, subject in rows:
        if ns >= last:
            break
        if event == "iter_start":
            continue
        if event.endswith("_start"):
            opened.add((resource, event[:-6], subject))
        elif event.endswith("_end"):
            opened.discard((resource, event[:-4], subject))
    out = [(0, r, k + "_start", s + " prev") for r, k, s in sorted(opened)]
    carried = set(opened)
    for ns, resource, event, subject in rows:
        if ns < last or event == "iter_start":
            continue
        if event.endswith("_end") and (resource, event[:-4], subject) in carried:
            carried.discard((resource, event[:-4], subject))
            subject += " prev"
        out.append((ns - last, resource, event, subject))
    return out


def summarize(rows) -> dict:
    """Per-resource busy time (union of start/end intervals), the end of the
    last forward / backward compute event, and per-chunk start times of
    uploads, offloads and host updates (first occurrence)."""
    open_at: dict = {}
    intervals: dict[str, list] = {}
    firsts: dict[str, dict] = {}
    fwd_end = bwd_end = 0
    end = 0
    for ns, resource, event, subject in rows:
        end = max(end, ns)
        if event.endswith("_start"):
            open_at[(resource, event[:-6], subject)] = ns
            kind = event[:-6]
            if kind in ("upload", "offload", "update", "optim"):
                firsts.setdefault(kind, {}).setdefault(subject, ns)
        elif event.endswith("_end"):
            kind = event[:-4]
            start = open_at.pop((resource, kind, subject), None)
            if start is not None:
                intervals.setdefault(resource, []).append((start, ns))
            if kind == "fwd":
                fwd_end = max(fwd_end, ns)
            if kind == "bwd":
                bwd_end = max(bwd_end, ns)
    busy = {}
    for resource, iv in intervals.items():
        iv.sort()
        tot, cur_s, cur_e = 0, None, None
        for s, e in iv:
            if cur_e is None or s > cur_e:
                if cur_e is not None:
                    tot += cur_e - cur_s
                cur_s, cur_e = s, e
            else:
                cur_e = max(cur_e, e)
        if cur_e is not None:
            tot += cur_e - cur_s
        busy[resource] = tot
    return {"end_ns": end, "fwd_end_ns": fwd_end, "bwd_end_ns": bwd_end, "busy_ns": busy,
            "first_start_ns": firsts}
