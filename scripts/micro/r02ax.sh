#!/bin/bash
# round 2 (ax): CTA-0 tile traces of the MXFP4 GEMM at HEAD on the Llama-3.2-1B K = 2048 shapes:
# single accumulator (product rule for K < 4096) vs overlapping double accumulators, with and
# without the epilogue's staging + stores (GEMM_ABLATE 8|32)
OUT=gpurun_out/${1:-r02ax}; mkdir -p $OUT
for shape in "16384 8192 2048" "16384 2048 2048" "16384 2048 8192"; do
  for ovl in 0 1; do
    for lib in gtr gtr_nostore; do
      echo "== $shape ovl=$ovl lib=$lib" >> $OUT/trace.txt
      ADAHOP_GEMM_OVL=$ovl ADAHOP_LIB=$PWD/build_variants/libadahop_$lib.so timeout 120 python scripts/micro/gemm_trace.py $shape 2>&1 | tail -28 >> $OUT/trace.txt
    done
  done
done
for ovl in 0 1; do
  echo "== shapes ovl=$ovl" >> $OUT/shapes.txt
  ADAHOP_GEMM_OVL=$ovl ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py 1b >> $OUT/shapes.txt 2>&1
done
echo done > $OUT/DONE
