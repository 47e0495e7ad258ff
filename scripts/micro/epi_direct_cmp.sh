#!/bin/bash
OUT=gpurun_out/epidirect; mkdir -p $OUT
L=$PWD/paper_2604_02525_b200/libadahop_direct.so
ADAHOP_LIB=$L timeout 600 python -m pytest tests -m gpu -x -q -k "gemm or linear" > $OUT/pytest_direct.log 2>&1; echo "rc=$?" >> $OUT/pytest_direct.log
ADAHOP_LIB=$L timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/gemm_direct_1b.log 2>&1
timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/gemm_staged_1b.log 2>&1
ADAHOP_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-cublas > $OUT/bench_direct.log 2>&1
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-cublas > $OUT/bench_staged.log 2>&1
