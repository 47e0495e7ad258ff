#!/bin/bash
OUT=gpurun_out/foidrows; mkdir -p $OUT
for r in 1024 2048 4096; do
  ADAHOP_FOID_BLOCK_ROWS=$r timeout 600 python -m pytest tests -m gpu -x -q -k "foid or linear or adahop_gemm" > $OUT/pytest_$r.log 2>&1; echo "rc=$?" >> $OUT/pytest_$r.log
  ADAHOP_FOID_BLOCK_ROWS=$r timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-cublas > $OUT/bench_$r.log 2>&1
done
