#!/bin/bash
# round 2 (bp): band-counted slice copies, the slice job's columns re-read from L2 after the stage is released
OUT=gpurun_out/${1:-r02bp}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py tests/test_gpu_fullsize.py -q -x -rf > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
B="python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20"
for i in 1 2 3; do
  for v in 1 0; do
    echo "== bands $v" >> $OUT/ab.txt
    ADAHOP_OR_BANDS=$v ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 $B 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stages_ms_per_step'], {k: (v['adahop_ms'], v['stages_ms']['quant']) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
  done
done
echo done > $OUT/DONE
