#!/bin/bash
# round 2 (ay): paced epilogue stores (ADAHOP_GEMM_PACE cycles per k-step between box stores) on the 1B GEMM shapes
OUT=gpurun_out/${1:-r02ay}; mkdir -p $OUT
for pace in 0 16 24 32 40 48; do
  echo "== pace $pace" >> $OUT/shapes.txt
  ADAHOP_GEMM_PACE=$pace ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py 1b 2>&1 | grep -v -i warn >> $OUT/shapes.txt
  echo "== pace $pace" >> $OUT/trace.txt
  ADAHOP_GEMM_PACE=$pace ADAHOP_LIB=$PWD/build_variants/libadahop_gtr.so timeout 120 python scripts/micro/gemm_trace.py 16384 8192 2048 2>&1 | tail -28 >> $OUT/trace.txt
done
echo done > $OUT/DONE
