#!/bin/bash
# round 2 (ao): with TMA-store epilogues, the 256x128 double-buffered tiles vs 256x256 per shape (short K)
OUT=gpurun_out/r02ao; mkdir -p $OUT
for v in 256 128 256 128; do
  for m in 1b 8b; do
    echo "== variant $v $m" >> $OUT/variants.txt
    ADAHOP_GEMM_VARIANT=$v ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py $m 2>&1 | grep -v -i warn >> $OUT/variants.txt
  done
done
