#!/bin/bash
# overlapping double accumulators: parity subset, per-shape A/B vs the single accumulator, tile trace
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm or linear" > $OUT/pytest_gemm.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gemm.txt
for o in 1 0; do
  echo "== ovl $o" >> $OUT/ab.txt
  ADAHOP_GEMM_OVL=$o ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py 1b 2>&1 | grep -v -i warn >> $OUT/ab.txt
  ADAHOP_GEMM_OVL=$o ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_exp.so timeout 300 python scripts/micro/gemm_cluster_bench.py 8b 2>&1 | grep -v -i warn >> $OUT/ab.txt
done
for s in "16384 8192 2048" "16384 2048 8192"; do
  echo "== $s" >> $OUT/trace.txt
  ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_gtr.so timeout 120 python scripts/micro/gemm_trace.py $s 2>&1 | tail -12 >> $OUT/trace.txt
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench.txt 2>&1
