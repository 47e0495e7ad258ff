#!/bin/bash
# round 2 (u): in-kernel X column gather (gather-by-MMA) feeding the fused outlier product: GPU suite,
# racecheck of the small workload, A/B vs the separate gather launch
OUT=gpurun_out/r02u; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python scripts/sanitize_layer.py > $OUT/sanitizer_racecheck.txt 2>&1; echo "rc=$?" >> $OUT/sanitizer_racecheck.txt
for f in 1 0 1 0; do
  echo "== ADAHOP_CG=$f" >> $OUT/cg_ab.txt
  ADAHOP_CG=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/cg_ab.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split > $OUT/ncu_launch.log 2>&1
