#!/bin/bash
# round 2 (w): short-K (epilogue / HBM-write bound) MXFP4 GEMMs: 1-CTA 128x128 kernel vs CTA pairs, tile traces
OUT=gpurun_out/r02w; mkdir -p $OUT
for v in 1 256; do
  for m in 1b 8b; do
    echo "== variant $v $m" >> $OUT/variants.txt
    ADAHOP_GEMM_VARIANT=$v ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py $m 2>&1 | grep -v -i warn >> $OUT/variants.txt
  done
done
for o in 0 1; do
  echo "== trace 16384 2048 512 ovl $o" >> $OUT/trace.txt
  ADAHOP_GEMM_OVL=$o ADAHOP_LIB=$PWD/build_variants/libadahop_gtr.so timeout 120 python scripts/micro/gemm_trace.py 16384 2048 512 2>&1 | tail -10 >> $OUT/trace.txt
done
