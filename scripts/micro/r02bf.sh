#!/bin/bash
# round 2 (bf): BF16 GEMM on CTA pairs (Lv2 CC) — parity, Instella-3B Lv2 and 1B Lv2 steps vs the 1-CTA kernel
OUT=gpurun_out/${1:-r02bf}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_split.py -q -x -rf > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for i in 1 2; do
  for v in pair onecta; do
    case $v in
      pair) E="";;
      onecta) E="ADAHOP_BF16_2SM=0";;
    esac
    for w in "instella_3b" "llama32_1b"; do
      echo "== $v $w lv2" >> $OUT/ab.txt
      env $E ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --workload $w --level 2 --no-e2e --no-cpu-baseline --no-split --steps 10 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['speedup_vs_cublas_bf16'],3), d['stages_ms_per_step'], {k: (v['adahop_ms'], round(v['speedup'],2)) for k, v in d['per_linear'].items()})" >> $OUT/ab.txt
    done
  done
done
echo done > $OUT/DONE
