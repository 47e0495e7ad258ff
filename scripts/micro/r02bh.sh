#!/bin/bash
# round 2 (bh): CTA-0 tile traces of the small 1B GEMM shapes (k / v fwd and dgrad) with store pacing
OUT=gpurun_out/${1:-r02bh}; mkdir -p $OUT
for shape in "16384 512 2048" "16384 2048 512" "16384 2048 2048"; do
  for ovl in 0 1; do
    echo "== $shape ovl=$ovl" >> $OUT/trace.txt
    ADAHOP_GEMM_OVL=$ovl ADAHOP_LIB=$PWD/build_variants/libadahop_gtr.so timeout 120 python scripts/micro/gemm_trace.py $shape 2>&1 | tail -30 >> $OUT/trace.txt
  done
done
echo done > $OUT/DONE
