#!/bin/bash
# round 2 (af): FOID + column gather in one launch (k_foid_gather_cols): GPU suite, A/B vs keys + select + gather
OUT=gpurun_out/r02af; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
for f in 1 0 1 0; do
  echo "== ADAHOP_FOID_GATHER=$f" >> $OUT/fg_ab.txt
  ADAHOP_FOID_GATHER=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/fg_ab.txt
done
