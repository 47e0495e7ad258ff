#!/bin/bash
# round 2 (ac): accumulator rule in the step with TMA-store epilogues: default (overlap for K >= 4096), overlap everywhere, single everywhere
OUT=gpurun_out/r02ac; mkdir -p $OUT
for o in -1 1 0 -1 1 0; do
  echo "== ADAHOP_GEMM_OVL=$o" >> $OUT/ovl_ab.txt
  ADAHOP_GEMM_OVL=$o ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/ovl_ab.txt
done
for o in -1 1 0; do
  echo "== 8b ADAHOP_GEMM_OVL=$o" >> $OUT/ovl_ab.txt
  ADAHOP_GEMM_OVL=$o ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --workload llama3_8b --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 10 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/ovl_ab.txt
done
