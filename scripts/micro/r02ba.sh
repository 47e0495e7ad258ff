#!/bin/bash
# round 2 (ba): paced epilogue stores, pace x min(nks, 8) cycles per box, last tile unpaced: per shape
# (1B, 8B) and in the layer step
OUT=gpurun_out/${1:-r02ba}; mkdir -p $OUT
for pace in 0 24 28 32 36; do
  for m in 1b 8b; do
    echo "== pace $pace $m" >> $OUT/shapes.txt
    ADAHOP_GEMM_PACE=$pace ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py $m 2>&1 | grep -v -i warn >> $OUT/shapes.txt
  done
done
B="python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20"
for i in 1 2 3; do
  for pace in 0 28 32; do
    echo "== step pace $pace" >> $OUT/ab.txt
    ADAHOP_GEMM_PACE=$pace ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'])" >> $OUT/ab.txt
  done
done
echo done > $OUT/DONE
