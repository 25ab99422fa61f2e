#!/bin/bash
# Compare the chunk-Adam kernel shapes on cfg2 on ONE box: parity of each,
# then ROUNDS interleaved bench passes (box / power-state drift hits every
# variant equally). Set NCU=1 for a full ncu capture of NCU_VARIANTS.
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/variants.jsonl
VARS=${VARIANTS:-tma1536x8t384 tma1536x8t384h tma1536x9t384 tma1536x9t384h tma1536x4x2t384 tma2048x6 tma2048x6h tma1792x7t448 ldg}
for v in $VARS; do
  PTK_ADAM_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_adam.py -x -q -m gpu -k "bit_exact or nonfinite" > $OUT/pytest_$v.log 2>&1
  echo "$v parity rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
for r in $(seq ${ROUNDS:-2}); do
  for v in $VARS; do
    PTK_ADAM_VARIANT=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --train-steps 0 --steps 50 > $OUT/bench_$v.json 2>$OUT/bench_$v.err
    python -c "import json;d=json.load(open('$OUT/bench_$v.json'));r=d['roofline'];print(json.dumps({'variant':'$v','round':$r,'step_gbs':d['value'],'kernel_gbs':r['achieved'],'frac':r['frac'],'live_copy':r['live_copy_gbs_this_box'],'frac_live':r['frac_of_live_copy'],'sm_mhz':d['clocks']['sm_mhz'],'reasons':d['clocks']['reasons']}))" | tee -a $OUT/variants.jsonl
  done
done
if [ "${NCU:-0}" = "1" ]; then
for v in ${NCU_VARIANTS:-tma1536x8t384}; do
PTK_ADAM_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:chunk_adam_tma -s 2 -c 1 \
  -o $OUT/prof_adam_$v -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --train-steps 0 > $OUT/ncu_$v.log 2>&1; echo "ncu $v rc=$?"
done
fi
