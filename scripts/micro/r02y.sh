#!/bin/bash
# round 2 (y): bench lines at HEAD — configs[1] layer (default), Llama-3-8B layer, config-5 stack with
# calibration -> plan, per-path API, Instella-3B; reference arm; ncu launch lists + full captures
OUT=gpurun_out/r02y; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
cp gpurun_out/bench_per_gemm.json $OUT/bench_per_gemm.json 2>/dev/null
timeout 900 python bench.py --workload llama3_8b --no-cpu-baseline --steps 5 > $OUT/bench_8b.log 2>&1
timeout 900 python bench.py --workload instella_3b --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_instella.log 2>&1
timeout 900 python bench.py --per-path --no-cpu-baseline --no-e2e --no-split --steps 10 > $OUT/bench_per_path.log 2>&1
timeout 1500 python bench.py --workload llama32_1b_stack --steps 5 --warmup 3 > $OUT/bench_stack.log 2>&1; echo "rc=$?" >> $OUT/bench_stack.log
cp gpurun_out/plan_llama32_1b_stack.json $OUT/ 2>/dev/null
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.log 2>&1
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv $NCUB > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches_8b.csv $NCUB --workload llama3_8b > $OUT/ncu_launch_bench_8b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_mxf4_2sm -s 12 -c 1 \
  -o $OUT/gemm $NCUB > $OUT/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_quant_tc -s 4 -c 1 \
  -o $OUT/quant $NCUB > $OUT/ncu_quant.log 2>&1
echo done > $OUT/DONE
