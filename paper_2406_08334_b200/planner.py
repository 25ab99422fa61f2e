"""Python access to the chunk planner (layouts for the data plane).

The planner is the C++ drop-in of the reference API (include/memplan/*.hpp,
built as build/memplan); `layout_for` returns the `pack` JSON of a named
workload trace: {"s_chunk", "n_chunk", "waste_bytes", "chunks": [...],
"bytes_per_param"}.
"""
from __future__ import annotations

import json
import os
import subprocess
import tempfile

from . import REPO_DIR

MEMPLAN_BIN = os.path.join(REPO_DIR, "build", "memplan")
GOLDEN_DIR = os.path.join(REPO_DIR, "tests", "golden")

# named traces: gen-trace arguments
TRACE_ARGS = {
    "gpt2-1b_b2": ["--model", "gpt2-1b", "--batch", "2"],
    "gpt2-1.5b_b8": ["--spec", os.path.join(GOLDEN_DIR, "gpt2_1.5b_spec.json"), "--batch", "8"],
    "gpt2-10b_b8": ["--model", "gpt2-10b", "--batch", "8"],
    "llama-13b_b8": ["--model", "llama-13b", "--batch", "8"],
}


def run_memplan(args: list[str]) -> str:
    if not os.path.exists(MEMPLAN_BIN):
        raise FileNotFoundError(f"{MEMPLAN_BIN} not built: run `make planner`")
    r = subprocess.run([MEMPLAN_BIN] + args, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"memplan {' '.join(args)} failed ({r.returncode}): {r.stderr.strip()}")
    return r.stdout


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
    """Chunk layout of a named trace, produced by the clean-room planner
    (raises if build/memplan is missing: no fallback to stored layouts)."""
    return _with_trace(name, pack)
