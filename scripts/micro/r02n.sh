#!/bin/bash
# round 2 (n): wgrad OE-Right outlier product fused into k_quant_tc: GPU suite, A/B vs the BF16 outlier GEMM
OUT=gpurun_out/r02n; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
for f in 1 0 1 0; do
  echo "== ADAHOP_OR_FUSED=$f" >> $OUT/or_ab.txt
  ADAHOP_OR_FUSED=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/or_ab.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split > $OUT/ncu_launch.log 2>&1
