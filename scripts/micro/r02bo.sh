#!/bin/bash
# round 2 (bo): ncu --set full of the gate fwd GEMM at HEAD (9th MXFP4 GEMM launch of the step now that k / v are grouped)
OUT=gpurun_out/${1:-r02bo}; mkdir -p $OUT
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_mxf4_2sm -s 8 -c 1 -o $OUT/gemm $NCUB > $OUT/ncu_gemm.log 2>&1
echo done > $OUT/DONE
