#!/bin/bash
OUT=gpurun_out/r02e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_parity.py -q -rf -k "split or extreme or context" > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
timeout 900 python bench.py > $OUT/bench.txt 2>&1; echo "rc=$?" >> $OUT/bench.txt
cp gpurun_out/bench_per_gemm.json $OUT/ 2>/dev/null
