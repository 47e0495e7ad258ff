for a in 0 1 2 3 4 7; do
  if [ $a = 0 ]; then L=paper_2604_02525_b200/libadahop.so; else L=paper_2604_02525_b200/libadahop_a$a.so; fi
  ADAHOP_LIB=$PWD/$L ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/abl_$a.csv python scripts/quant_microbench.py 16384x8192,16384x2048 > /dev/null 2>&1
done
