#!/bin/bash
# round 2 (v): MXFP4 GEMM variant per shape: 256x128 double-buffered (128) vs 256x256 single / overlapping accumulators
OUT=gpurun_out/r02v; mkdir -p $OUT
for cfg in "256 -1" "128 -1" "256 1" "256 0"; do
  set -- $cfg
  for m in 1b 8b; do
    echo "== variant $1 ovl $2 $m" >> $OUT/variants.txt
    ADAHOP_GEMM_VARIANT=$1 ADAHOP_GEMM_OVL=$2 ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py $m 2>&1 | grep -v -i warn >> $OUT/variants.txt
  done
done
