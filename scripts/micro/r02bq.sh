#!/bin/bash
# round 2 (bq): no split-K inside the layer / split-step calls: full GPU suite, bench step
OUT=gpurun_out/${1:-r02bq}; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.txt 2>&1; echo "rc=$?" >> $OUT/bench.txt
timeout 900 python bench.py --workload llama3_8b --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_8b.txt 2>&1
echo done > $OUT/DONE
