"""Python access to the chunk planner (layouts for the data plane).

The planner is the C++ drop-in of the reference API (include/memplan/*.hpp),
linked into libptk.so and called IN PROCESS through the C-ABI
(ptk_memplan_run = memplan::run_cli, proj/include/memplan/cli.hpp:20-35): no
subprocess, no binary on PATH. `layout_for` returns the `pack` JSON of a named
workload trace: {"s_chunk", "n_chunk", "waste_bytes", "chunks": [...],
"bytes_per_param"}.
"""
from __future__ import annotations

import json
import os
import tempfile

from . import REPO_DIR

GOLDEN_DIR = os.path.join(REPO_DIR, "tests", "golden")

# named traces: gen-trace arguments
TRACE_ARGS = {
    "gpt2-1b_b2": ["--model", "gpt2-1b", "--batch", "2"],
    "gpt2-1.5b_b8": ["--spec", os.path.join(GOLDEN_DIR, "gpt2_1.5b_spec.json"), "--batch", "8"],
    "gpt2-10b_b8": ["--model", "gpt2-10b", "--batch", "8"],
    "llama-13b_b8": ["--model", "llama-13b", "--batch", "8"],
}


def run_memplan(args: list[str]) -> str:
    """One memplan command in process; raises with its stderr on a nonzero exit."""
    from . import _native
    rc, out, err = _native.memplan_run(args)
    if rc != 0:
        raise RuntimeError(f"memplan {' '.join(args)} failed ({rc}): {err.strip()}")
    return out


def trace_file(args: list[str], path: str) -> str:
    """Synthesize a trace with the planner (`memplan gen-trace`)."""
    run_memplan(["gen-trace"] + args + ["-o", path])
    return path


def _with_trace(name: str, fn):
    """Run fn(trace_path) on a freshly generated trace in a private scratch
    directory: concurrent ranks of one job never share (or race on) a file."""
    with tempfile.TemporaryDirectory(prefix="ptk_planner_") as d:
        return fn(trace_file(TRACE_ARGS[name], os.path.join(d, f"trace_{name}.json")))


def trace_for(name: str) -> dict:
    def load(path):
        with open(path) as f:
            return json.load(f)
    return _with_trace(name, load)


def pack(trace_path: str, grid: str | None = None) -> dict:
    out = json.loads(run_memplan(["pack", "--trace", trace_path] + (["--grid", grid] if grid else [])))
    out.setdefault("bytes_per_param", 2)
    return out


def layout_for(name: str) -> dict:
    """Chunk layout of a named trace, produced by the planner in libptk.so
    (raises if the library is missing: no fallback to stored layouts)."""
    return _with_trace(name, pack)
