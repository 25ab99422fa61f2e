#!/bin/bash
# round-2 profiling pass: launch list of the default bench, ncu --set full of the
# chunk-table Adam (cfg2 and the 93-chunk cfg2x32 table) and of the fused TMA
# kernel (W=4, 512 MiB, virtual ranks), fused virtual-rank timing, N=2 self-launch flow
cd "$(dirname "$0")/.."
OUT=gpurun_out/${TAG:-r02p}; mkdir -p $OUT
B="python bench.py --steps 2 --warmup 3 --train-steps 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv \
  $B > $OUT/ncu_list.log 2>&1; echo "ncu-list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chunk_adam_tma -s 2 -c 1 \
  -o $OUT/prof_adam_cfg2 -f $B --no-e2e > $OUT/ncu_adam_cfg2.log 2>&1; echo "ncu-adam-cfg2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chunk_adam_tma -s 2 -c 1 \
  -o $OUT/prof_adam_cfg2x32 -f $B --no-e2e --workload cfg2x32 > $OUT/ncu_adam_cfg2x32.log 2>&1; echo "ncu-adam-x32 rc=$?"
for c in "512 1" "32 16" "32 1"; do set -- $c
  timeout 600 python scripts/fused_virtual_bench.py --chunk-mib $1 --chunks $2 --worlds 1,2,4,8 2>&1 | tail -4
  PTK_FUSED_KERNEL=ldg timeout 600 python scripts/fused_virtual_bench.py --chunk-mib $1 --chunks $2 --worlds 2,4,8 2>&1 | tail -3
done
cp gpurun_out/fused_virtual.jsonl $OUT/ 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_peer_tma -s 4 -c 1 \
  -o $OUT/prof_fused_w4 -f python scripts/fused_virtual_bench.py --chunk-mib 512 --worlds 4 --steps 1 --warmup 1 \
  > $OUT/ncu_fused_w4.log 2>&1; echo "ncu-fused rc=$?"
timeout 600 python bench.py --gpus 2 --shared-device --steps 5 --warmup 3 --train-steps 0 --no-cpu-baseline \
  > $OUT/bench_shared2.json 2> $OUT/bench_shared2.err; echo "shared2 rc=$?"; tail -c 1500 $OUT/bench_shared2.json; tail -3 $OUT/bench_shared2.err
