"""The chunk runtime (memplan::execute via ptk_execute_plan) executes a plan
with the simulator's decisions and real bytes; its measured timeline is
checked against the simulator's for the same plan.

With enough buffers there is no eviction, so the runtime's chunk lifecycle is
fully determined: every non-persistent chunk is uploaded exactly once before
its forward, reduced -> offloaded -> updated on the host exactly once after
its backward, every persistent chunk gets one device Adam, and each swap
block streams all its activation-holding ops out and back in. The event
multiset must then equal the simulator's (times differ: they are measured),
byte counters must equal the real shard / activation sizes, and causal order
must hold per chunk (upload_end < first fwd_start of the chunk; offload after
the chunk's last bwd_end; update after offload).
"""
import collections
import ctypes
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MEMPLAN = os.path.join(REPO, "build", "memplan")

PROFILE = {"h2d_bw": 5.0e10, "d2h_bw": 5.0e10, "coll_alpha": 2e-5, "coll_bw": 7.0e11,
           "world_size": 1, "gpu_mem": 180_000_000_000, "cpu_mem": 1_000_000_000_000,
           "cpu_optim_rate": 1.0e9, "gpu_optim_rate": 5.0e10}


def _files(tmp_path, np_=None, nb=None, ns=0, nc=0):
    """Trace (6-block GPT-2 shape), 32 MiB chunk layout, a bare PlanConfig
    (np_/nb None = all persistent / all buffered), the simulator's timeline."""
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"hidden_size": 1024, "n_blocks": 6, "n_heads": 16,
                                "vocab_size": 8192, "seq_len": 512}))
    trace = str(tmp_path / "trace.json")
    subprocess.run([MEMPLAN, "gen-trace", "--spec", str(spec), "--batch", "4", "-o", trace],
                   check=True)
    prof = tmp_path / "hw.json"
    prof.write_text(json.dumps(PROFILE))
    plan = str(tmp_path / "plan.json")
    layout = json.loads(subprocess.run([MEMPLAN, "pack", "--trace", trace, "--grid", "32Mi"],
                                       check=True, capture_output=True, text=True).stdout)
    n = layout["n_chunk"]
    np_ = n if np_ is None else np_
    nb = n - np_ if nb is None else nb
    cfg = {"s_chunk": 32 << 20, "n_chunk": n, "n_persist": np_, "n_buffer": nb,
           "n_block": 6, "n_interval": 1, "n_swap": ns, "n_checkpoint": nc}
    with open(plan, "w") as f:
        json.dump(cfg, f)
    sim_csv = tmp_path / "sim.csv"
    subprocess.run([MEMPLAN, "simulate", "--trace", trace, "--hw", str(prof), "--plan", plan,
                    "--timeline-csv", str(sim_csv)], check=True, capture_output=True)
    sim = [tuple(line.split(",", 3)) for line in sim_csv.read_text().splitlines()[1:]]
    return trace, plan, str(prof), layout, sim


def _events(tl):
    return collections.Counter((r, e, s.strip('"')) for _, r, e, s in tl)


@pytest.mark.parametrize("np_,ns,nc", [(1, 0, 0), (0, 1, 2), (2, 0, 3)])
def test_executor_matches_simulated_lifecycle(tmp_path, cuda_device, np_, ns, nc):
    from paper_2406_08334_b200 import runtime
    # n_buffer = every non-persistent chunk keeps its buffer: no eviction
    trace, plan, prof, layout, sim = _files(tmp_path, np_, None, ns, nc)
    n = layout["n_chunk"]
    res = runtime.execute_plan(trace, plan, prof, compute_scale=1.0, iterations=2)
    ours = _events(res["timeline"])
    theirs = collections.Counter((r, e, s.strip('"')) for _, r, e, s in sim)
    assert ours == theirs
    # real bytes: one upload + one offload of every non-persistent shard
    shards = [c["used_bytes"] for c in layout["chunks"][np_:]]
    pad = [(b // 2 + 7) // 8 * 8 * 2 for b in shards]
    tr = json.load(open(trace))
    swap_bytes = sum(op["act_bytes"] for op in tr["ops"]
                     if op["block_id"] is not None and op["block_id"] < ns * 2 and
                     op["block_id"] % 2 == 0) if ns else 0
    assert res["h2d_bytes"] == sum(pad) + swap_bytes
    assert res["d2h_bytes"] == sum(pad) + swap_bytes
    # causality per chunk
    first = {}
    for t, r, e, s in res["timeline"]:
        first.setdefault((r, e, s.strip('"')), t)
    for c in range(np_ + 1, n + 1):
        tag = f"chunk={c}"
        assert first[("h2d", "upload_end", tag)] <= first[("d2h", "offload_start", tag)]
        assert first[("d2h", "offload_end", tag)] <= first[("cpu", "update_start", tag)]
    # the measured iteration cannot beat its own compute
    compute = sum(op["t_fwd"] + op["t_bwd"] for op in tr["ops"])
    assert res["t_iter"] >= 0.98 * compute
    assert res["t_iter"] <= 3.0 * res["estimate_t_iter"] + 0.05


def test_compute_bound_plan_matches_estimate(tmp_path, cuda_device):
    """All persistent, compute dominates: measured t_iter ~ estimate."""
    from paper_2406_08334_b200 import runtime
    trace, plan, prof, layout, sim = _files(tmp_path)
    res = runtime.execute_plan(trace, plan, prof, compute_scale=1.0, iterations=2)
    rel = abs(res["t_iter"] - res["estimate_t_iter"]) / res["estimate_t_iter"]
    assert rel < 0.15, res


def test_measured_profile_is_sane(tmp_path, cuda_device):
    from paper_2406_08334_b200 import runtime
    base = tmp_path / "base.json"
    base.write_text(json.dumps(PROFILE))
    hw = runtime.measure_profile(str(base), str(tmp_path / "b200x1.json"))
    assert 5e9 < hw["h2d_bw"] < 2e11 and 5e9 < hw["d2h_bw"] < 2e11
    assert hw["gpu_optim_rate"] > 5e10      # >= 1.4 TB/s of 28 B/param
    assert hw["cpu_optim_rate"] > 1e7
    assert hw["gpu_mem"] > 100e9
    # the individual ptk_profile_* probes agree with the composed profile's ranges
    from paper_2406_08334_b200 import _native as nat
    h2d, d2h, rate = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    nat.lib.ptk_profile_copy_bw(64 << 20, ctypes.byref(h2d), ctypes.byref(d2h))
    assert 5e9 < h2d.value < 2e11 and 5e9 < d2h.value < 2e11
    nat.lib.ptk_profile_gpu_adam_rate(64 << 20, ctypes.byref(rate))
    assert rate.value > 5e10
    subprocess.run([MEMPLAN, "list-presets"], check=True, capture_output=True)


def test_host_memory_bandwidth_probe():
    """ptk_profile_host_memory_bw (the simulator's --host-mem-bw input): host
    Adam + concurrent pinned copies, a positive bandwidth of a plausible size,
    and argument checks that fail loudly."""
    import ctypes
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200 import runtime
    bw = runtime.host_memory_bw(n=4 << 20, seconds=0.3)
    assert 1e9 < bw < 5e12
    out = ctypes.c_double()
    assert nat.raw.ptk_profile_host_memory_bw(0, 0, 0.3, ctypes.byref(out)) != nat.PTK_OK
    assert "ptk_profile_host_memory_bw" in nat.last_error()
