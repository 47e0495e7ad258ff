#!/bin/bash
# round 2 (be): row-streaming column gather for narrow tensors vs the per-element gather
OUT=gpurun_out/${1:-r02be}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -rf > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
B="python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20"
for i in 1 2 3; do
  for v in prod nostream; do
    case $v in
      prod) L=$PWD/paper_2604_02525_b200/libadahop.so; E="";;
      nostream) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_GATHER_STREAM=0";;
    esac
    echo "== $v" >> $OUT/ab.txt
    env $E ADAHOP_LIB=$L timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'], {k: (v['adahop_ms'], v['stages_ms']['quant']) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
  done
done
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv $NCUB > $OUT/ncu_launch.log 2>&1
echo done > $OUT/DONE
