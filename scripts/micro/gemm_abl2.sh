#!/bin/bash
OUT=gpurun_out/abl2; mkdir -p $OUT
./build_micro/tmem_ld_bw > $OUT/tmem_ld_bw.log 2>&1
for a in 0 1 2 4 8 10; do
  if [ $a = 0 ]; then L=paper_2604_02525_b200/libadahop.so; else L=paper_2604_02525_b200/libadahop_g$a.so; fi
  ADAHOP_LIB=$PWD/$L timeout 300 python scripts/micro/gemm_cluster_bench.py 1b > $OUT/abl_$a.log 2>&1
done
ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_tr.so timeout 300 python scripts/micro/gemm_trace.py > $OUT/trace.log 2>&1
