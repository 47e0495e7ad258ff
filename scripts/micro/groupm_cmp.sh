#!/bin/bash
OUT=gpurun_out/groupm; mkdir -p $OUT
for g in 4 8 16; do
  if [ $g = 8 ]; then L=paper_2604_02525_b200/libadahop.so; else L=paper_2604_02525_b200/libadahop_g$g.so; fi
  ADAHOP_LIB=$PWD/$L timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/g${g}_1b.log 2>&1
  ADAHOP_LIB=$PWD/$L timeout 300 python scripts/micro/gemm_cluster_bench.py 8b > $OUT/g${g}_8b.log 2>&1
done
