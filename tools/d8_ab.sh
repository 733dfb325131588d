make -C paper_2605_13928_b200/csrc -j16 > /dev/null 2>&1
for r in 1 2; do for n in base h4 m6 h4m6 m8; do
  if [ $n = base ]; then L=; else L=$PWD/paper_2605_13928_b200/libscb_b200_$n.so; fi
  echo -n "$n "; SCB_LIB_PATH=$L timeout 300 python tools/delta8_time.py 2>&1 | tail -1
done; done
