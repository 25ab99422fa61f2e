#!/bin/bash
# cfg5 chunk-size sweep (flat 32-512 MiB chunks) + cfg1 on one GPU.
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/sweep.jsonl
for w in flat32 flat64 flat128 flat256 flat512 cfg1 cfg2; do
  timeout 300 python bench.py --workload $w --steps ${STEPS:-200} --warmup 5 --no-cpu-baseline ${EXTRA:-} >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
  echo "$w rc=$?"
done
python - <<'PY'
import json
for line in open("gpurun_out/sweep.jsonl"):
    d = json.loads(line)
    print(d["config"]["workload"].split(":")[0], d["value"], d["ms_per_step"], d["roofline"]["achieved"],
          d["roofline"]["frac"], (d.get("e2e") or {}).get("value"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
