#!/bin/bash
# config 4: Llama-3-8B layer step with OE k in {0, 16, 64}; full-size layer parity tests
OUT=gpurun_out/ksweep; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > $OUT/pytest_fullsize.log 2>&1; echo "rc=$?" >> $OUT/pytest_fullsize.log
for k in 0 16 64; do
  timeout 600 python bench.py --workload llama3_8b --oe-k $k --steps 5 --no-e2e --no-cpu-baseline > $OUT/bench_8b_k$k.log 2>&1
done
