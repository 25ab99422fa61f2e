#!/bin/bash
# compute-sanitizer over every libptk kernel at test sizes (race
# detection / memory checking is new in this build). memcheck on the kernel
# and chunk-step parity tests; racecheck + synccheck on a focused driver that
# launches each kernel once (shared-memory hazards of the TMA ring, barrier
# misuse). Logs land in gpurun_out/sanitize_*.log.
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='bit_exact or nonfinite or stats or gscale or virtual or nccl_mode or clipping or skips or pinned'
echo "== memcheck"
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_gpu_adam.py tests/test_gpu_chunkset.py -q -m gpu -k "$SEL" \
  > $OUT/sanitize_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitize_memcheck.log | tail -3
for tool in racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_driver.py \
    > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|driver ok" $OUT/sanitize_$tool.log | tail -2
done
