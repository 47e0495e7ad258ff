#!/bin/bash
# parity + timing of the MXFP4 GEMM for each cluster shape (ADAHOP_GEMM_CLUSTER)
OUT=gpurun_out/gemm_cluster
mkdir -p $OUT
for c in 1 2 4 21 22; do
  ADAHOP_GEMM_CLUSTER=$c timeout 300 python -m pytest tests -m gpu -x -q -k "gemm or linear" > $OUT/pytest_$c.log 2>&1
  echo "cluster $c rc=$?" >> $OUT/pytest_$c.log
  ADAHOP_GEMM_CLUSTER=$c timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/bench1b_$c.log 2>&1
  ADAHOP_GEMM_CLUSTER=$c timeout 300 python scripts/micro/gemm_cluster_bench.py 8b > $OUT/bench8b_$c.log 2>&1
done
