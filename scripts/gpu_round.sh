#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines, ncu launch list and full captures.
# Usage (from this container): gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh [tag] [quick]'
set -u
TAG=${1:-r01}
MODE=${2:-full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
if [ $MODE = full ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
fi
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
cp gpurun_out/bench_per_gemm.json $OUT/bench_per_gemm.json 2>/dev/null
timeout 600 python bench.py --workload llama3_8b --no-cpu-baseline --steps 5 > $OUT/bench_8b.log 2>&1
if [ $MODE = full ]; then
  timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.log 2>&1
fi
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph"
# launch list of one step (cold-cache, serialised) with DRAM bytes per launch
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv $NCUB > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches_8b.csv $NCUB --workload llama3_8b > $OUT/ncu_launch_bench_8b.log 2>&1
if [ $MODE = full ]; then
  # full captures: the gate-projection fwd GEMM (13th GEMM launch of the step) and its quant launch (5th)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_mxf4_2sm -s 12 -c 1 \
    -o $OUT/gemm $NCUB > $OUT/ncu_gemm.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_quant_tc -s 4 -c 1 \
    -o $OUT/quant $NCUB > $OUT/ncu_quant.log 2>&1
fi
echo done > $OUT/DONE
# multi-rank plumbing smoke on one GPU (gloo; NCCL needs one GPU per rank): the torchrun path
ADAHOP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 \
  > $OUT/two_rank_gloo.log 2>&1; echo "rc=$?" >> $OUT/two_rank_gloo.log
