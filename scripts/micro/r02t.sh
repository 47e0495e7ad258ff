#!/bin/bash
# round 2 (t): compute-sanitizer evidence (memcheck / racecheck / synccheck) on a small layer workload,
# then the default bench line and an ncu launch list at HEAD
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 120 python scripts/sanitize_layer.py > $OUT/plain.txt 2>&1; echo "rc=$?" >> $OUT/plain.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_layer.py > $OUT/sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> $OUT/sanitizer_$tool.txt
done
timeout 900 python bench.py > $OUT/bench.txt 2>&1; echo "rc=$?" >> $OUT/bench.txt
cp gpurun_out/bench_per_gemm.json $OUT/ 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split > $OUT/ncu_launch.log 2>&1
