#!/bin/bash
# round 2 (bl): a small linear's MXFP4 GEMMs in one grouped persistent launch vs separate launches
OUT=gpurun_out/${1:-r02bl}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x -rf > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
B="python bench.py --no-e2e --no-cpu-baseline --no-split --steps 20"
for i in 1 2; do
  for g in 1 0; do
    for w in llama32_1b llama3_8b instella_3b; do
      echo "== group $g $w" >> $OUT/ab.txt
      ADAHOP_GEMM_GROUP=$g ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 $B --workload $w 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['speedup_vs_cublas_bf16'],3), d['stages_ms_per_step'], {k: (v['adahop_ms'], round(v['speedup'],2)) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
    done
  done
done
echo done > $OUT/DONE
