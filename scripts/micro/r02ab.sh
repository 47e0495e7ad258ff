#!/bin/bash
# round 2 (ab): MXFP4 GEMM epilogue by TMA stores (128B-swizzled 32-row boxes) vs LSU stores; with it,
# the overlapping accumulators on every K; GPU suite on the product build
OUT=gpurun_out/r02ab; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
for cfg in "1 -1" "0 -1" "1 1" "1 0"; do
  set -- $cfg
  echo "== tma_store $1 ovl $2" >> $OUT/gemm.txt
  ADAHOP_GEMM_TMA_STORE=$1 ADAHOP_GEMM_OVL=$2 ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py 1b 2>&1 | grep -v -i warn >> $OUT/gemm.txt
done
for f in 1 0 1 0; do
  echo "== ADAHOP_GEMM_TMA_STORE=$f" >> $OUT/step_ab.txt
  ADAHOP_GEMM_TMA_STORE=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/step_ab.txt
done
