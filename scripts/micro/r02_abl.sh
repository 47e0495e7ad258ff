#!/bin/bash
# GEMM ablations: which part bounds the main loop (A/B feed, scale factors, MMA issue, stores)
OUT=gpurun_out/r02b; mkdir -p $OUT
for a in 0 16 21 5 8; do
  if [ $a = 0 ]; then L=paper_2604_02525_b200/libadahop.so; else L=paper_2604_02525_b200/libadahop_g$a.so; fi
  echo "== ablate $a" >> $OUT/abl.txt
  ADAHOP_LIB=$PWD/$L timeout 300 python scripts/micro/gemm_cluster_bench.py 1b 2>&1 | grep -v Warn | grep -v warn_once >> $OUT/abl.txt
done
for s in "16384 8192 2048" "16384 2048 8192"; do
  echo "== notrace-ablate16 $s" >> $OUT/trace16.txt
  ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_gtr16.so timeout 120 python scripts/micro/gemm_trace.py $s 2>&1 | tail -12 >> $OUT/trace16.txt
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> $OUT/smi.txt
