#!/bin/bash
# round 2 (bb): store pacing slot = pace x min(nks, 16) (exp) vs min(nks, 8) (exp8): per shape and in the steps
OUT=gpurun_out/${1:-r02bb}; mkdir -p $OUT
for v in exp exp8; do
  for pace in 28 32; do
    for m in 1b 8b; do
      echo "== $v pace $pace $m" >> $OUT/shapes.txt
      ADAHOP_GEMM_PACE=$pace ADAHOP_LIB=$PWD/build_variants/libadahop_$v.so timeout 300 python scripts/micro/gemm_cluster_bench.py $m 2>&1 | grep -v -i warn >> $OUT/shapes.txt
    done
  done
done
B="python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20"
for i in 1 2; do
  for cfg in "exp 0" "exp 30" "exp8 30" "exp 34"; do
    set -- $cfg
    for m in llama32_1b llama3_8b; do
      echo "== step $1 pace $2 $m" >> $OUT/ab.txt
      ADAHOP_GEMM_PACE=$2 ADAHOP_LIB=$PWD/build_variants/libadahop_$1.so timeout 600 $B --workload $m 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'])" >> $OUT/ab.txt
    done
  done
done
echo done > $OUT/DONE
