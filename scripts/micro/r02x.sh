#!/bin/bash
# round 2 (x): how much of the bf16 GEMM epilogue's cost is smem staging vs global stores
OUT=gpurun_out/r02x; mkdir -p $OUT
for a in 0 8 32 0; do
  if [ $a = 0 ]; then L=$PWD/paper_2604_02525_b200/libadahop.so; else L=$PWD/build_variants/libadahop_g$a.so; fi
  echo "== ablate $a" >> $OUT/abl.txt
  ADAHOP_LIB=$L timeout 300 python scripts/micro/gemm_cluster_bench.py 1b 2>&1 | grep -v -i warn >> $OUT/abl.txt
done
