#!/bin/bash
# round 2 (s): where the fused outlier product's quant-stage cost comes from:
# 1 fused, 0 BF16 GEMM, 2 fused-kernel variant without product (single TMEM buffer, 3 stages), 3 OR tile order without product
OUT=gpurun_out/r02s; mkdir -p $OUT
for f in 1 0 2 3 1 0 2 3; do
  echo "== ADAHOP_OR_FUSED=$f" >> $OUT/or_ab.txt
  ADAHOP_OR_FUSED=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/or_ab.txt
done
