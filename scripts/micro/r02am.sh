#!/bin/bash
# round 2 (am): OE-Left wgrad product fused too (1) vs OE-Right only (4), layer step and per linear
OUT=gpurun_out/r02am; mkdir -p $OUT
for f in 1 4 1 4; do
  echo "== ADAHOP_OR_FUSED=$f" >> $OUT/or_ab.txt
  ADAHOP_OR_FUSED=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'], {k: v['adahop_ms'] for k, v in (d.get('per_linear') or {}).items()})" >> $OUT/or_ab.txt
done
