#!/bin/bash
# round 2 (bm): validation with the grouped-launch rule: pytest -m gpu, smoke, bench lines, launch list, step A/B
OUT=gpurun_out/${1:-r02bm}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.txt 2>&1; echo "rc=$?" >> $OUT/bench.txt
timeout 900 python bench.py --workload llama3_8b --no-cpu-baseline --steps 5 > $OUT/bench_8b.txt 2>&1
timeout 900 python bench.py --workload instella_3b --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_instella.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20"
for i in 1 2; do
  for g in 1 0; do
    echo "== group $g" >> $OUT/ab.txt
    ADAHOP_GEMM_GROUP=$g ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['speedup_vs_cublas_bf16'],3), d['stages_ms_per_step'], {k: (v['adahop_ms'], round(v['speedup'],2)) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
  done
done
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv $NCUB > $OUT/ncu_launch.log 2>&1
echo done > $OUT/DONE
