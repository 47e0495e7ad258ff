#!/bin/bash
OUT=gpurun_out/overlap2; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for n in 1 0; do
  ADAHOP_OVERLAP=$n timeout 600 python bench.py --no-e2e --no-cpu-baseline > $OUT/bench_1b_$n.log 2>&1
  ADAHOP_OVERLAP=$n timeout 600 python bench.py --workload llama3_8b --steps 5 --no-e2e --no-cpu-baseline > $OUT/bench_8b_$n.log 2>&1
done
