for l in 1 2 3 4; do
  ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_l$l.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_mxf4 --csv --log-file gpurun_out/gl_$l.csv python scripts/micro/gemm_shapes.py > /dev/null 2>&1
done
