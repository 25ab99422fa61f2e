#!/bin/bash
# One GPU-box pass: tests, smoke, bench, ncu launch list + full capture of the
# dominant kernel. Everything lands in gpurun_out/ (merged back by gpurun).
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
echo "== pytest -m gpu"; timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
echo "== bench"; timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json; tail -3 $OUT/bench.err
if [ "${NCU:-1}" = "1" ]; then
# the chunk-step phase of the bench only (no e2e / training / CPU baseline)
NCU_BENCH="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --train-steps 0"
echo "== ncu launch list"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  $NCU_BENCH > $OUT/ncu_launch_bench.log 2>&1; echo "ncu-list rc=$?"
echo "== ncu full"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:chunk_adam_tma -s 2 -c 1 \
  -o $OUT/prof_adam -f $NCU_BENCH > $OUT/ncu_full.log 2>&1; echo "ncu-full rc=$?"
fi
echo done
