#!/bin/bash
OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_plan.py -q -rf > $OUT/pytest_plan.txt 2>&1; echo "rc=$?" >> $OUT/pytest_plan.txt
timeout 1500 python bench.py --workload llama32_1b_stack --steps 5 --warmup 3 > $OUT/bench_stack.txt 2>&1; echo "rc=$?" >> $OUT/bench_stack.txt
cp gpurun_out/plan_llama32_1b_stack.json $OUT/ 2>/dev/null
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $OUT/smi.txt
