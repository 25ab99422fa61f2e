"""Run under torchrun (CPU, gloo): each rank starts bench.py's child-job
mechanism (_run_child) with the trivial `--leg ping` and prints the result."""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

world, rank, local = bench.dist_setup()
sys.argv = [sys.argv[0], "--gpus", str(world)]
res, err = bench._run_child(types.SimpleNamespace(), world, rank, local, ["--leg", "ping"], 120, "ping")
with open(os.path.join(os.environ["PROBE_OUT_DIR"], f"rank{rank}.json"), "w") as f:
    json.dump({"rank": rank, "res": res, "err": err}, f)
