#!/bin/bash
# round 2 (z): FOID launches with PDL (A/B), the GEMM-alone entry point test, the bench line with our GEMMs timed beside cuBLASLt
OUT=gpurun_out/r02z; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "gemm" > $OUT/pytest_gemm.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gemm.txt
for f in 0 1 2 0 1 2; do
  echo "== ADAHOP_FOID_PDL=$f" >> $OUT/foid_pdl.txt
  ADAHOP_FOID_PDL=$f ADAHOP_LIB=$PWD/build_variants/libadahop_exp.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-split --no-cublas --steps 20 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'], d['ms_per_step_instrumented'])" >> $OUT/foid_pdl.txt
done
timeout 900 python bench.py --no-e2e --no-cpu-baseline > $OUT/bench.txt 2>&1
