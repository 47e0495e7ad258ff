#!/bin/bash
# round 2 (ar): split-K cluster GEMM per shape (forced 2 / 4 pairs, auto, off), split-K tile trace,
# layer-step A/B (product vs no split-K vs lane=row column gather)
OUT=gpurun_out/${1:-r02ar}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "gemm or layer or outlier or oe" > $OUT/pytest_gemm.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gemm.txt
for s in 1 0 2 4; do
  ADAHOP_GEMM_SPLITK=$s ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/gemm_splitk_bench.py >> $OUT/splitk_shapes.txt 2>&1
done
for s in 2 4; do
  echo "== trace split $s" >> $OUT/trace.txt
  ADAHOP_GEMM_SPLITK=$s ADAHOP_LIB=$PWD/build_variants/libadahop_gtr.so timeout 120 python scripts/micro/gemm_trace.py 512 2048 16384 >> $OUT/trace.txt 2>&1
done
echo "== trace 256x128" >> $OUT/trace.txt
ADAHOP_GEMM_SPLITK=0 ADAHOP_LIB=$PWD/build_variants/libadahop_gtr.so timeout 120 python scripts/micro/gemm_trace.py 512 2048 16384 >> $OUT/trace.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20"
for i in 1 2; do
  for v in prod nosplit oldgather; do
    case $v in
      prod) L=$PWD/paper_2604_02525_b200/libadahop.so; E="";;
      nosplit) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_GEMM_SPLITK=0";;
      oldgather) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_GATHER_COLS=0";;
    esac
    echo "== $v" >> $OUT/ab.txt
    env $E ADAHOP_LIB=$L timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'], {k: (v['adahop_ms'], v['stages_ms']['gemm_mxf4'], v['stages_ms']['quant'], v['stages_ms']['outlier']) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
  done
done
echo done > $OUT/DONE
