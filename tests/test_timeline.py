"""CPU tests of the measured-timeline helpers (paper_2406_08334_b200.timeline):
CSV round trip in the simulator's schema, the last-iteration cut with
carried-over intervals, busy-time union."""
from paper_2406_08334_b200.timeline import last_iteration, read_csv, summarize, write_csv


ROWS = [(0, "gpu", "iter_start", "iter=0"), (5, "cpu", "update_start", "chunk=3"),
        (10, "gpu", "iter_start", "iter=1"), (12, "cpu", "update_end", "chunk=3"),
        (13, "gpu", "fwd_start", "block=0"), (20, "gpu", "fwd_end", "block=0"),
        (15, "h2d", "upload_start", "chunk=2"), (18, "h2d", "upload_end", "chunk=2"),
        (21, "gpu", "bwd_start", "block=0"), (30, "gpu", "bwd_end", "block=0")]


def test_last_iteration_rebases_and_marks_carried_intervals():
    rows = sorted(ROWS)
    tail = last_iteration(rows)
    assert tail[0] == (0, "cpu", "update_start", "chunk=3 prev")
    assert (2, "cpu", "update_end", "chunk=3 prev") in tail
    assert (3, "gpu", "fwd_start", "block=0") in tail
    assert all(e != "iter_start" for _, _, e, _ in tail)
    assert last_iteration([(1, "gpu", "fwd_start", "block=0")]) == [(1, "gpu", "fwd_start",
                                                                     "block=0")]


def test_summary_and_csv_round_trip(tmp_path):
    tail = last_iteration(sorted(ROWS))
    s = summarize(tail)
    assert s["fwd_end_ns"] == 10 and s["bwd_end_ns"] == 20 and s["end_ns"] == 20
    assert s["busy_ns"]["gpu"] == (10 - 3) + (20 - 11)
    assert s["busy_ns"]["h2d"] == 3 and s["busy_ns"]["cpu"] == 2
    assert s["first_start_ns"]["upload"] == {"chunk=2": 5}
    p = str(tmp_path / "t.csv")
    write_csv(tail, p)
    assert read_csv(p) == tail


def test_chrome_trace_matches_the_simulators_format(tmp_path):
    """write_chrome_trace of a timeline equals, event for event, what the
    planner writes for the same timeline (`memplan simulate --timeline`,
    read back through its `--timeline-csv`)."""
    import json

    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.timeline import write_chrome_trace
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"hidden_size": 256, "n_blocks": 4, "n_heads": 4,
                                "vocab_size": 1000, "seq_len": 128}))
    tpath = planner.trace_file(["--spec", str(spec), "--batch", "4"], str(tmp_path / "t.json"))
    sim_chrome, sim_csv = tmp_path / "sim.json", tmp_path / "sim.csv"
    planner.run_memplan(["simulate", "--trace", tpath, "--hw", "a100x1", "--s-chunk", "4194304",
                         "--n-persist", "1", "--n-buffer", "1", "--timeline", str(sim_chrome),
                         "--timeline-csv", str(sim_csv)])
    rows = read_csv(str(sim_csv))
    assert len(rows) > 10
    ours = tmp_path / "ours.json"
    write_chrome_trace(rows, str(ours))
    assert json.loads(ours.read_text()) == json.loads(sim_chrome.read_text())
