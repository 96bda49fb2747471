for rep in 1 2 3; do
for v in base tswap; do
  if [ $v = base ]; then L=""; else L=_ab/$v.so; fi
  DMQR_LIB_PATH=$L timeout 200 python tools/ab_time.py 4096 5 2>&1 | sed "s/^/$v /"
done; done
