#!/bin/bash
# round 2 (br): the dgrad OE-Left product fused into W's quant pass (second fused product per launch)
OUT=gpurun_out/${1:-r02br}; mkdir -p $OUT
timeout 300 python scripts/micro/dgrad_or_debug.py > $OUT/debug.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
B="python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20"
for i in 1 2; do
  for v in 1 0; do
    for w in llama32_1b llama3_8b; do
      echo "== dgrad-fused $v $w" >> $OUT/ab.txt
      ADAHOP_OR_DGRAD=$v ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 $B --workload $w 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['speedup_vs_cublas_bf16'],3), d['stages_ms_per_step'], {k: (v['adahop_ms'], round(v['speedup'],2)) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
    done
  done
done
echo done > $OUT/DONE
