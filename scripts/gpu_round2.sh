#!/bin/bash
# multicast probe, host memory, graph-timed chunk-size sweep, large-model training with measured plans
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 60 ./build/probe_multicast > $OUT/probe_mc.txt 2>&1; cat $OUT/probe_mc.txt
(free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; nproc; ulimit -l) > $OUT/host_mem.txt 2>&1; cat $OUT/host_mem.txt
STEPS=200 bash scripts/sweep.sh 2>&1 | tail -8
for m in ${MODELS:-llama-13b gpt2-10b}; do
  echo "== train_large $m"
  timeout 1500 python scripts/train_large.py --model $m --batch 8 > $OUT/train_large_$m.log 2>&1; echo "rc=$?"
  tail -c 3000 $OUT/train_large_$m.log
done
