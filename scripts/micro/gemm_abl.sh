for a in 0 1 2 4 8 3 5; do
  if [ $a = 0 ]; then L=paper_2604_02525_b200/libadahop.so; else L=paper_2604_02525_b200/libadahop_g$a.so; fi
  ADAHOP_LIB=$PWD/$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_mxf4 --csv --log-file gpurun_out/ga_$a.csv python scripts/micro/gemm_shapes.py > /dev/null 2>&1
done
