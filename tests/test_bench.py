"""bench.py's contract on CPU: `--gpus N` self-launches N ranks under
torch.distributed.run (the reference arm runs on rank 0 and reports
n_gpus = N), a WORLD_SIZE / --gpus mismatch fails loudly, and the byte counts
behind `value` and the roofline equal BASELINE.md §3's table."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402


def _last_json(stdout: str) -> dict:
    for line in reversed(stdout.strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise AssertionError(f"no JSON line in: {stdout[-2000:]}")


def test_self_launch_reference_arm_two_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--workload", "flat32", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "torch.distributed.run" in r.stderr  # went through the self-launch
    d = _last_json(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["parallelism"] == "zero3-dp2" and d["same_config"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
    assert "memplan_plan_s" in d["cpu_baseline"]["extras"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    # exactly one JSON line: rank 1 exits without printing
    assert sum(1 for line in r.stdout.splitlines() if line.startswith("{")) == 1


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--workload", "flat32"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=REPO)
    assert r.returncode != 0
    assert "WORLD_SIZE=3" in r.stderr


FLAT512 = [(512 << 20) // 2]
CFG2 = [512_420_800, 522_593_600, 522_593_600]


@pytest.mark.parametrize("numels,w,hbm_gb,nvl_gb", [
    (FLAT512, 1, 7.516, 0.0),
    (FLAT512, 8, 2.013, 0.940),
    ([(32 << 20) // 2], 8, 0.126, 0.059),
    (CFG2, 1, 43.613, 0.0),
    (CFG2, 8, 11.682, 5.452),
])
def test_metric_bytes_match_baseline_table(numels, w, hbm_gb, nvl_gb):
    assert round(bench.metric_hbm_bytes(numels, w) / 1e9, 3) == hbm_gb
    assert round(bench.nvlink_bytes(numels, w) / 1e9, 3) == nvl_gb


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_fused_kernel_bytes_and_bound(w):
    """The fused launch moves 28P/w + 4P(w-1)/w HBM bytes and 4P(w-1)/w
    NVLink bytes per direction per rank (not 2P(w-1)/w); w >= 4 is NVLink-bound."""
    p = FLAT512[0]
    hbm, nvl = bench.dominant_kernel_bytes(FLAT512, w, "fused")
    assert hbm == 28 * p // w + 4 * p * (w - 1) // w
    assert nvl == 4 * p * (w - 1) // w
    k = {"kernel": "x", "ms": 1.0, "hbm_bytes": hbm, "nvl_bytes": nvl, "launches": 1,
         "chunks_per_launch": 1, "world": w, "timing": "t"}
    roof = bench.roofline(k, 6457.4, "measured", "flat512")
    want_nvl = nvl / bench.NVLINK_GBS > hbm / 6457.4
    assert roof["bound"] == ("nvlink" if want_nvl else "hbm")
    if w >= 4:
        assert roof["bound"] == "nvlink"
        assert roof["achieved"] == round(nvl / 1e-3 / 1e9, 1)
    # the NCCL leg's dominant kernel is the chunk-table Adam on the owned shard
    assert bench.dominant_kernel_bytes(FLAT512, w, "nccl") == (28 * p // w, 0)


def test_split_workloads_cover_cfg2():
    for mib in (32, 64, 128, 256, 512):
        numels, _ = bench.chunk_numels(f"cfg2x{mib}")
        assert sum(numels) == bench.CFG2_PARAMS
        assert max(numels) == (mib << 20) // 2
    assert len(bench.chunk_numels("cfg2x32")[0]) == 93


def test_child_job_under_torchrun(tmp_path):
    """The guarded child jobs of the N>1 legs (training, fused exchange):
    under torchrun each rank starts a child that forms its own group on a
    fresh port -- not on torchrun's agent store -- and hands back a result."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["PROBE_OUT_DIR"] = str(tmp_path)
    port = _free_port_cpu()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1", f"--master-port={port}",
                        os.path.join(REPO, "tests", "_child_probe.py")],
                       capture_output=True, text=True, timeout=300, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    got = [json.loads((tmp_path / f"rank{q}.json").read_text()) for q in range(2)]
    assert [d["res"] for d in got] == [{"rank": 0, "world": 2}, {"rank": 1, "world": 2}], got


def _free_port_cpu():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,piece,up,down", [(512_420_800, 1 << 25, True, True),
                                             (522_593_600, 1 << 25, False, True),
                                             (1 << 21, 1 << 25, True, True),
                                             (3 << 20, 1 << 20, True, False)])
def test_e2e_pieces_cover_the_chunk(n, piece, up, down):
    got = bench.e2e_pieces(n, piece, up, down)
    assert got[0][0] == 0 and sum(m for _, m in got) == n
    assert all(lo % 8 == 0 for lo, _ in got)
    assert all(a[0] + a[1] == b[0] for a, b in zip(got, got[1:]))
    if up and n > 4 * piece:
        assert got[0][1] == 1 << 20
    if down and n > 4 * piece:
        assert got[-1][1] == 1 << 20


def test_reference_arm_line_n1():
    """--impl reference at N=1: the oracle port of the same step on the host
    cores, same metric / unit / config keys as the GPU arm, e2e = the line's
    own value with no host<->device bytes."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                        "--workload", "flat32", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["unit"] == "GB/s"
    assert d["metric"] == bench.METRIC and d["higher_is_better"] is True
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["same_config"] is True
