#!/bin/bash
# round 2 (bi): ncu --set full of the FOID keys and select kernels (2048 stored rows, strided probe; 16384 contiguous)
OUT=gpurun_out/${1:-r02bi}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_foid -s 6 -c 4 -o $OUT/foid python scripts/micro/foid_graph_time.py > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
