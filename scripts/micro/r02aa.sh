#!/bin/bash
# round 2 (aa): TMA issue from several lanes of one warp (micro) and k_quant_tc with two issuing lanes (A/B)
OUT=gpurun_out/r02aa; mkdir -p $OUT
timeout 120 ./build_micro/tma_feed2 > $OUT/tma_feed2.txt 2>&1
for v in exp q2 exp q2; do
  echo "== $v" >> $OUT/q2_ab.txt
  ADAHOP_LIB=$PWD/build_variants/libadahop_$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/q2_ab.txt
done
