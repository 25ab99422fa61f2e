#!/bin/bash
# round-2 GPU check: the GPU test suite, smoke, default bench, chunk-size sweep (table launch)
cd "$(dirname "$0")/.."
OUT=gpurun_out/${TAG:-r02}; mkdir -p $OUT
nvidia-smi -L; free -g | head -2; nproc
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_ARGS} > $OUT/pytest.log 2>&1; echo "pytest rc=$?"
tail -40 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke.log
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err; echo "bench rc=$?"
tail -c 2500 $OUT/bench_cfg2.json; tail -5 $OUT/bench_cfg2.err
for w in ${SWEEP:-cfg2x32 cfg2x64 cfg2x128 cfg2x256 cfg2x512 flat32 flat512}; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --train-steps 0 --no-cpu-baseline > $OUT/sweep_$w.json 2> $OUT/sweep_$w.err
  python -c "import json,sys; d=json.load(open('$OUT/sweep_$w.json')); r=d['roofline']; print('$w', d['value'], d['ms_per_step'], r['frac'], r['ms_per_launch'], r['chunks_per_launch'])" || tail -5 $OUT/sweep_$w.err
done
fi
