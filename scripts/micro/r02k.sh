#!/bin/bash
# round 2 (k): TMA feed micro (producers vs bytes in flight), quant OE-mask A/B (bitmap vs index list)
OUT=gpurun_out/r02k; mkdir -p $OUT
timeout 120 ./build_micro/tma_feed2 > $OUT/tma_feed2.txt 2>&1; echo "rc=$?" >> $OUT/tma_feed2.txt
for v in cur bitmap cur bitmap; do
  if [ $v = cur ]; then L=$PWD/paper_2604_02525_b200/libadahop.so; else L=$PWD/build_variants/libadahop_bitmap.so; fi
  echo "== $v" >> $OUT/mask_ab.txt
  ADAHOP_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/mask_ab.txt
done
