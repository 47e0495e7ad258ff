#!/bin/bash
# round 2 (aw): FOID in one cluster launch (no index divisions, ~1024 rows per CTA) and the fused
# product's slice copied in-kernel with band counters (no gather launch): parity, micro, step A/B
OUT=gpurun_out/${1:-r02aw}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x -rf > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
timeout 300 python scripts/micro/foid_graph_time.py > $OUT/foid_micro_prod.txt 2>&1
ADAHOP_FOID_CLUSTER=0 ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 300 python scripts/micro/foid_graph_time.py > $OUT/foid_micro_2launch.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20"
for i in 1 2 3; do
  for v in prod nobands nofoidc neither; do
    case $v in
      prod) L=$PWD/paper_2604_02525_b200/libadahop.so; E="";;
      nobands) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_OR_BANDS=0";;
      nofoidc) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_FOID_CLUSTER=0";;
      neither) L=$PWD/build_variants/libadahop_exp.so; E="ADAHOP_FOID_CLUSTER=0 ADAHOP_OR_BANDS=0";;
    esac
    echo "== $v" >> $OUT/ab.txt
    env $E ADAHOP_LIB=$L timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'], {k: (v['adahop_ms'], v['stages_ms']['foid'], v['stages_ms']['quant']) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
  done
done
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv $NCUB > $OUT/ncu_launch.log 2>&1
echo done > $OUT/DONE
