#!/bin/bash
# round 2 (bu): final validation at HEAD (dgrad product fused, grouped launch, pacing, BF16 pair GEMM): pytest -m gpu, smoke, every bench line, ncu launch lists + full captures, two ranks on one GPU
OUT=gpurun_out/r02bu; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.txt 2>&1; echo "rc=$?" >> $OUT/bench.txt
cp gpurun_out/bench_per_gemm.json $OUT/ 2>/dev/null
timeout 900 python bench.py --workload llama3_8b --no-cpu-baseline --steps 5 > $OUT/bench_8b.txt 2>&1
timeout 900 python bench.py --workload instella_3b --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_instella.txt 2>&1
timeout 900 python bench.py --workload instella_3b --level 2 --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_instella_lv2.txt 2>&1
timeout 900 python bench.py --per-path --no-cpu-baseline --no-e2e --no-split --steps 10 > $OUT/bench_per_path.txt 2>&1
for k in 0 16; do timeout 900 python bench.py --workload llama3_8b --oe-k $k --no-cpu-baseline --no-e2e --no-split --steps 5 > $OUT/bench_8b_k$k.txt 2>&1; done
timeout 1500 python bench.py --workload llama32_1b_stack --steps 5 --warmup 3 --adaptive-k > $OUT/bench_stack_adaptive.txt 2>&1
timeout 1500 python bench.py --workload llama32_1b_stack --steps 5 --warmup 3 > $OUT/bench_stack.txt 2>&1
cp gpurun_out/plan_llama32_1b_stack.json $OUT/ 2>/dev/null
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.txt 2>&1
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv $NCUB > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches_8b.csv $NCUB --workload llama3_8b > $OUT/ncu_launch_8b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_mxf4_2sm -s 8 -c 1 -o $OUT/gemm $NCUB > $OUT/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_quant_tc -s 4 -c 1 -o $OUT/quant $NCUB > $OUT/ncu_quant.log 2>&1
ADAHOP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 > $OUT/two_rank_gloo.txt 2>&1; echo "rc=$?" >> $OUT/two_rank_gloo.txt
echo done > $OUT/DONE
