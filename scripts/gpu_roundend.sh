#!/bin/bash
# What the driver runs at round end, in its order: the GPU test suite, smoke(),
# the reference arm, then the bench line (N=1).
cd "$(dirname "$0")/.."
OUT=gpurun_out/${TAG:-roundend}; mkdir -p $OUT
timeout 1800 python -m pytest tests -x -q -m gpu --timeout 900 > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps ${K:-20} --warmup ${W:-5} > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"; tail -c 600 $OUT/ref.json; tail -3 $OUT/ref.err
timeout 900 python bench.py --gpus 1 --steps ${K:-20} --warmup ${W:-5} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err
python - <<'PY'
import json, os
out = os.environ.get("OUT_DIR", "gpurun_out/" + os.environ.get("TAG", "roundend"))
d = json.load(open(out + "/bench.json")); r = json.load(open(out + "/ref.json"))
print("bench", d["value"], d["unit"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "launches", d["gpu_launches"], "clocks", d["clocks"])
print("ref", r["value"], r["unit"], "same_config", r["same_config"], "cores", r["cpu_baseline"]["cores"])
print("e2e / ref", round(d["e2e"]["value"] / r["value"], 3), "device / ref", round(d["value"] / r["value"], 2))
PY
