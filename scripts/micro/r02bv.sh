#!/bin/bash
# round 2 (bv): overlapping double accumulators on every shape (ADAHOP_GEMM_OVL=1) vs the rule (K >= 4096) now that stores are paced
OUT=gpurun_out/${1:-r02bv}; mkdir -p $OUT
for o in -1 1 0; do
  for m in 1b 8b; do
    echo "== ovl $o $m" >> $OUT/shapes.txt
    ADAHOP_GEMM_OVL=$o ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py $m 2>&1 | grep -v -i warn >> $OUT/shapes.txt
  done
done
B="python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20"
for i in 1 2 3; do
  for o in -1 1; do
    echo "== step ovl $o" >> $OUT/ab.txt
    ADAHOP_GEMM_OVL=$o ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'])" >> $OUT/ab.txt
  done
done
echo done > $OUT/DONE
