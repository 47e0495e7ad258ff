#!/bin/bash
# OE-slice gathers: separate launches (default) vs copied from the staged tiles inside k_quant_tc
OUT=gpurun_out/r02f; mkdir -p $OUT
for f in 0 1 0 1; do
  echo "== ADAHOP_GATHER_FUSED=$f" >> $OUT/gather_ab.txt
  ADAHOP_GATHER_FUSED=$f ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/gather_ab.txt
done
# launch list of one step (product library, graph off so ncu sees every kernel)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-cublas --no-split --no-graph > $OUT/ncu_bench.log 2>&1
