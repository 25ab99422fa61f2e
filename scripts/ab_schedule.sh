#!/bin/bash
# A/B of the tile schedule (dynamic claim vs static round-robin) on the TMA kernels
cd "$(dirname "$0")/.."
OUT=gpurun_out/${TAG:-ab_sched}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "adam or chunkset or fused or smoke" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for rep in 1; do
for sched in dynamic static; do
  PTK_TILE_SCHEDULE=$sched timeout 600 python scripts/fused_virtual_bench.py --chunk-mib 512 --worlds 2,4,8 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l); print('$sched fused W=%d'%d['virtual_ranks'], d['ms_per_step'], d['frac'])
  except Exception: pass"
  for w in cfg2 cfg2x32 flat32 flat512; do
    PTK_TILE_SCHEDULE=$sched timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --train-steps 0 --no-cpu-baseline > $OUT/b_${sched}_$w.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/b_${sched}_$w.json')); r=d['roofline']; print('$sched adam $w', d['ms_per_step'], r['frac'])"
  done
done
done
