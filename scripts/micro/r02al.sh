#!/bin/bash
# round 2 (al): the wgrad OE-Left outlier product fused into X's quant pass (layer call): GPU suite, step A/B
OUT=gpurun_out/r02al; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
for f in 1 0 1 0; do
  echo "== ADAHOP_OR_FUSED=$f" >> $OUT/or_ab.txt
  ADAHOP_OR_FUSED=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'], {k: v['adahop_ms'] for k, v in (d.get('per_linear') or {}).items()})" >> $OUT/or_ab.txt
done
