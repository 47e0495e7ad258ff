for n in tr tr4 tr8; do
  echo "##### $n"
  ADAHOP_LIB=$PWD/paper_2604_02525_b200/libadahop_$n.so python scripts/micro/qtc_trace.py 2>&1 | grep -A40 "=== dual" | sed -n 30,36p
done
