#!/bin/bash
# round 2 (ai): outlier counts / adaptive k (DESIGN R16): GPU tests, then the config-5 stack with k = 64 vs adaptive k
OUT=gpurun_out/r02ai; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_plan.py -q -rf > $OUT/pytest_plan.txt 2>&1; echo "rc=$?" >> $OUT/pytest_plan.txt
timeout 1500 python bench.py --workload llama32_1b_stack --steps 5 --warmup 3 > $OUT/bench_stack_k64.txt 2>&1
timeout 1500 python bench.py --workload llama32_1b_stack --steps 5 --warmup 3 --adaptive-k > $OUT/bench_stack_adaptive.txt 2>&1
cp gpurun_out/plan_llama32_1b_stack.json $OUT/ 2>/dev/null
