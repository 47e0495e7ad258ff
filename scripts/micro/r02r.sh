#!/bin/bash
# round 2 (r): ncu full capture of the gate-projection quant launch, fused outlier product vs not
OUT=gpurun_out/r02r; mkdir -p $OUT
NCUB="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-graph --no-split"
for f in 1 0; do
  ADAHOP_OR_FUSED=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_quant_tc -s 4 -c 1 \
    -o $OUT/quant_or$f $NCUB > $OUT/ncu_quant_or$f.log 2>&1
done
