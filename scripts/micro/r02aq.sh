#!/bin/bash
# round 2 (aq): split-K clusters for long-K few-tile MXFP4 GEMMs, row-local column gather, direct-Dt
# BF16 outlier GEMM for short K: parity tests first, then A/B against the experiment build's knobs
OUT=gpurun_out/r02aq; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "gemm or layer" > $OUT/pytest_gemm.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gemm.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
B="python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20"
for i in 1 2 3; do
  for v in prod nosplit oldgather; do
    case $v in
      prod) L=$PWD/paper_2604_02525_b200/libadahop.so; E="";;
      nosplit) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_GEMM_SPLITK=0";;
      oldgather) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_GATHER_COLS=0";;
    esac
    echo "== $v" >> $OUT/ab.txt
    env $E ADAHOP_LIB=$L timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'], {k: v['adahop_ms'] for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
  done
done
timeout 900 python bench.py > $OUT/bench.txt 2>&1; echo "rc=$?" >> $OUT/bench.txt
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv $NCUB > $OUT/ncu_launch.log 2>&1
echo done > $OUT/DONE
