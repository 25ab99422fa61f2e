"""Python access to the chunk runtime (memplan::execute) and the profiler
re-feed (memplan::measure_profile), both in libptk.so behind the C-ABI
(include/ptk.h: ptk_execute_plan, ptk_measure_profile).

    result = execute_plan(trace, plan, profile, compute_scale=1.0, iterations=2)
    result["t_iter"], result["estimate_t_iter"], result["timeline"]  # measured

`measure_profile` writes a HardwareProfile JSON measured on this machine; feed
it to `memplan plan --hw <file>` to re-plan with measured rates.
"""
from __future__ import annotations

import csv
import io
import json
import os
import tempfile

from . import _native as nat


def execute_plan(trace_path: str, plan_path: str, profile_path: str, comm=None, rank: int = 0,
                 compute_scale: float = 1.0, iterations: int = 1) -> dict:
    with tempfile.TemporaryDirectory() as d:
        res, tl = os.path.join(d, "result.json"), os.path.join(d, "timeline.csv")
        nat.lib.ptk_execute_plan(trace_path.encode(), plan_path.encode(), profile_path.encode(),
                                 comm, rank, compute_scale, iterations, res.encode(), tl.encode())
        with open(res) as f:
            out = json.load(f)
        with open(tl) as f:
            out["timeline_csv"] = f.read()
    out["timeline"] = [(int(r["time_ns"]), r["resource"], r["event"], r["subject"])
                       for r in csv.DictReader(io.StringIO(out["timeline_csv"]))]
    return out


def measure_profile(base_profile_path: str, out_path: str, comm=None, world: int = 1) -> dict:
    nat.lib.ptk_measure_profile(base_profile_path.encode(), comm, world, out_path.encode())
    with open(out_path) as f:
        return json.load(f)


def host_memory_bw(n: int = 32 << 20, threads: int = 0, seconds: float = 1.0) -> float:
    """Host-memory bandwidth shared by the host Adam and pinned PCIe copies
    (bytes/s), for `memplan simulate --host-mem-bw` (ptk_profile_host_memory_bw)."""
    import ctypes
    out = ctypes.c_double()
    nat.lib.ptk_profile_host_memory_bw(n, threads, seconds, ctypes.byref(out))
    return out.value
