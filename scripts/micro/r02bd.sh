#!/bin/bash
# round 2 (bd): CTA-0 tile timeline of the quant pass in the layer call (gate, q, k)
OUT=gpurun_out/${1:-r02bd}; mkdir -p $OUT
for l in gate q k down; do
  ADAHOP_LIB=$PWD/build_variants/libadahop_qtr.so timeout 120 python scripts/micro/qtc_layer_trace.py $l > $OUT/trace_$l.txt 2>&1
done
echo done > $OUT/DONE
