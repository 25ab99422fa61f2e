#!/bin/bash
# Compare the chunk-Adam kernel variants on cfg2 (bench) and check parity of each.
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
for v in ${VARIANTS:-tma1536x8t384 tma2048x6 tma1536x8t192 tma3072x4t384 tma1792x7t448 tma1536x9t384 tma1280x10t320 ldg}; do
  echo "== $v"
  PTK_ADAM_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_adam.py -x -q -m gpu -k "bit_exact or nonfinite" > $OUT/pytest_$v.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_$v.log
  PTK_ADAM_VARIANT=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 50 > $OUT/bench_$v.json 2>$OUT/bench_$v.err
  python -c "import json;d=json.load(open('$OUT/bench_$v.json'));print('$v', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['clocks'])"
done
if [ "${NCU:-0}" = "1" ]; then
for v in ${NCU_VARIANTS:-tma2048x6}; do
PTK_ADAM_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:chunk_adam_tma -s 2 -c 1 \
  -o $OUT/prof_adam_$v -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_$v.log 2>&1; echo "ncu $v rc=$?"
done
fi
