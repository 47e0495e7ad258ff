#!/bin/bash
# round 2 (ap): double-buffered TMEM for the plain tiles of a fused-product quant launch (db) vs single (sb)
OUT=gpurun_out/r02ap; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
for v in exp sb exp sb exp sb; do
  echo "== $v" >> $OUT/ab.txt
  ADAHOP_LIB=$PWD/build_variants/libadahop_$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/ab.txt
done
