"""CPU test of the full-depth trace expansion scripts/train_large.py feeds
the planner (BASELINE cfg3 / cfg4): the synthesized trace's operators and
parameter bytes, the profiled k-block model's measured values."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "scripts"))
MEMPLAN = os.path.join(REPO, "build", "memplan")


def _gen(tmp_path, name, args):
    p = str(tmp_path / name)
    subprocess.run([MEMPLAN, "gen-trace"] + args + ["-o", p], check=True)
    return json.load(open(p)), p


def test_expand_trace_replicates_measured_blocks(tmp_path):
    from train_large import expand_trace, spec_of
    from paper_2406_08334_b200.train import GPT2Shape
    full, _ = _gen(tmp_path, "full.json", ["--model", "llama-13b", "--batch", "8"])
    shape = GPT2Shape.from_trace(full)
    (tmp_path / "spec.json").write_text(json.dumps(spec_of(shape, 4)))
    small, _ = _gen(tmp_path, "small.json", ["--spec", str(tmp_path / "spec.json"), "--batch", "8"])
    # a stand-in "measurement": distinct values per operator and block
    meas = json.loads(json.dumps(small))
    for i, o in enumerate(meas["ops"]):
        b = o["block_id"] if o["block_id"] is not None else 0
        o.update(t_fwd=1e-3 * (i + 1), t_bwd=2e-3 * (i + 1) + b * 1e-6,
                 act_bytes=1000 * (i + 1), d_peak_op=7 * (i + 1))
    meas["m_fwd"] = 12345
    out = expand_trace(full, meas, 4, "test")
    assert [o["name"] for o in out["ops"]] == [o["name"] for o in full["ops"]]
    assert [o["param_bytes"] for o in out["ops"]] == [o["param_bytes"] for o in full["ops"]]
    assert out["n_blocks"] == full["n_blocks"] == 40 and out["m_fwd"] == 12345
    top = {o["name"]: o for o in meas["ops"] if o["block_id"] is None}
    for o in out["ops"]:
        if o["block_id"] is None:
            assert o["t_fwd"] == top[o["name"]]["t_fwd"]
        else:   # median over the 4 profiled blocks of the same operator kind
            kind = o["name"].split(".")[0]
            vals = sorted(m["t_bwd"] for m in meas["ops"] if m["name"].split(".")[0] == kind)
            assert o["t_bwd"] == (vals[1] + vals[2]) / 2
    # the planner accepts it
    path = tmp_path / "measured.json"
    path.write_text(json.dumps(out))
    r = subprocess.run([MEMPLAN, "pack", "--trace", str(path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["n_chunk"] == 40
