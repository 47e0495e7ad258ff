#!/bin/bash
# round 2 (i): TMA feed micro (second pass), quant stage with the warp-uniform OE mask, full GPU suite
OUT=gpurun_out/r02i; mkdir -p $OUT
timeout 120 ./build_micro/tma_feed2 > $OUT/tma_feed2.txt 2>&1; echo "rc=$?" >> $OUT/tma_feed2.txt
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 > $OUT/bench_quick.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
