#!/bin/bash
# Interleaved shape sweep of the chunk-Adam TMA kernel (bench build:
# -DPTK_BENCH_VARIANTS, build/ab/libptk_bench.so), one flat chunk of N params,
# per-launch GB/s at 28 B/param; the round-1 library (build/ab/libptk_old.so)
# as the reference point when present.
cd "$(dirname "$0")/.."
for N in ${NS:-268435456 16777216 522593600}; do
  REPS=$(( N < 50000000 ? 200 : 20 ))
  for round in 1 2; do
    for v in ${VARIANTS:-tma1536x9t384 tma2048x6t512 tma2048x6t512h tma2560x5t640 tma3072x4t768 tma1024x13t256 tma1792x7t448 tma1024x6x2t256}; do
      echo -n "$v "; PTK_ADAM_VARIANT=$v timeout 120 python scripts/ab_adam.py build/ab/libptk_bench.so $N $REPS
    done
    [ -f build/ab/libptk_old.so ] && { echo -n "r01 "; python scripts/ab_adam.py build/ab/libptk_old.so $N $REPS; }
  done
done
