#!/bin/bash
# round 2 (av): FOID in one launch (a cluster of CTAs per OE operand) vs keys + select launches
OUT=gpurun_out/${1:-r02av}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -q -x -rf > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
timeout 300 python scripts/micro/foid_graph_time.py > $OUT/foid_micro_prod.txt 2>&1
ADAHOP_FOID_CLUSTER=0 ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/foid_graph_time.py > $OUT/foid_micro_2launch.txt 2>&1
ADAHOP_FOID_PDL=1 ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/foid_graph_time.py > $OUT/foid_micro_pdl.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20"
for i in 1 2 3; do
  for v in prod twolaunch pdl; do
    case $v in
      prod) L=$PWD/paper_2604_02525_b200/libadahop.so; E="";;
      twolaunch) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_FOID_CLUSTER=0";;
      pdl) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_FOID_PDL=1";;
    esac
    echo "== $v" >> $OUT/ab.txt
    env $E ADAHOP_LIB=$L timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'], {k: (v['adahop_ms'], v['stages_ms']['foid']) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
  done
done
echo done > $OUT/DONE
