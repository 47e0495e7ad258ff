#!/bin/bash
# quick GPU check: gpu parity tests + the two bench lines (no ncu)
OUT=gpurun_out/${1:-quick}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
cp gpurun_out/bench_per_gemm.json $OUT/ 2>/dev/null
timeout 600 python bench.py --workload llama3_8b --no-cpu-baseline --steps 5 > $OUT/bench_8b.log 2>&1
