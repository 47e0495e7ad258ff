#!/bin/bash
OUT=gpurun_out/sfbmc; mkdir -p $OUT
L=$PWD/paper_2604_02525_b200/libadahop_sfbmc.so
ADAHOP_LIB=$L timeout 600 python -m pytest tests -m gpu -x -q -k "gemm or linear" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do
ADAHOP_LIB=$L timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/mc_1b_$i.log 2>&1
timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/base_1b_$i.log 2>&1
done
ADAHOP_LIB=$L timeout 300 python scripts/micro/gemm_cluster_bench.py 8b > $OUT/mc_8b.log 2>&1
timeout 300 python scripts/micro/gemm_cluster_bench.py 8b > $OUT/base_8b.log 2>&1
