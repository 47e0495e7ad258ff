#!/bin/bash
# round 2 (l): three TMA producer warps in the MXFP4 GEMM + per-launch OE bitmaps in k_quant_tc
OUT=gpurun_out/r02l; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf > $OUT/pytest_parity.txt 2>&1; echo "rc=$?" >> $OUT/pytest_parity.txt
timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/gemm_1b.txt 2>&1
timeout 300 python scripts/micro/gemm_cluster_bench.py 8b > $OUT/gemm_8b.txt 2>&1
for s in "16384 8192 2048" "16384 2048 8192"; do
  echo "== $s" >> $OUT/trace.txt
  ADAHOP_LIB=$PWD/build_variants/libadahop_gtr.so timeout 120 python scripts/micro/gemm_trace.py $s 2>&1 | tail -12 >> $OUT/trace.txt
done
for i in 1 2; do
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['speedup_vs_cublas_bf16'], d['stages_ms_per_step'], d['ms_per_step_instrumented'], d['roofline']['frac'])" >> $OUT/bench_quick.txt
done
