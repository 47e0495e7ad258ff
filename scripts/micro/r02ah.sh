#!/bin/bash
OUT=gpurun_out/r02ah; mkdir -p $OUT
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
ADAHOP_FOID_GATHER=1 ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $NCUB > $OUT/ncu_launch.log 2>&1
ADAHOP_FOID_GATHER=1 ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_foid_gather_cols -s 1 -c 1 -o $OUT/fg $NCUB > $OUT/ncu_fg.log 2>&1
