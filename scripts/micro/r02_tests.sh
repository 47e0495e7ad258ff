#!/bin/bash
OUT=gpurun_out/r02d; mkdir -p $OUT
timeout 120 ./build_micro/tma_feed > $OUT/tma_feed.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "rc=$?" >> $OUT/smoke.txt
