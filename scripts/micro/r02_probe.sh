#!/bin/bash
# round-2 probe: per-shape GEMM times, GEMM tile traces, TMA delivery rate
OUT=gpurun_out/r02a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/gemm_1b.txt 2>&1
timeout 300 python scripts/micro/gemm_cluster_bench.py 8b > $OUT/gemm_8b.txt 2>&1
for s in "16384 2048 2048" "16384 8192 2048" "16384 2048 8192" "2048 2048 16384"; do
  echo "== $s" >> $OUT/trace.txt
  ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_gtr.so timeout 120 python scripts/micro/gemm_trace.py $s 2>&1 | tail -24 >> $OUT/trace.txt
done
timeout 120 ./build_micro/tma_bw > $OUT/tma_bw.txt 2>&1
