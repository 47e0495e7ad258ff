#!/bin/bash
# round 2 (bk): quant pass: the column orientation's stores delayed after the row orientation's (QTC_STORE_PACE cycles)
OUT=gpurun_out/${1:-r02bk}; mkdir -p $OUT
B="python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20"
for i in 1 2 3; do
  for v in prod qsp600 qsp1200; do
    case $v in
      prod) L=$PWD/paper_2604_02525_b200/libadahop.so;;
      *) L=$PWD/build_variants/libadahop_$v.so;;
    esac
    echo "== $v" >> $OUT/ab.txt
    ADAHOP_LIB=$L timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'])" >> $OUT/ab.txt
  done
done
echo done > $OUT/DONE
