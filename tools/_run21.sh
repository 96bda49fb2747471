for rep in 1 2; do
for v in base colwarp prev; do
  if [ $v = base ]; then L=""; else L=_ab/$v.so; fi
  DMQR_LIB_PATH=$L timeout 200 python tools/ab_time.py 1024 3 cfg4 2>&1 | sed "s/^/$v /"
  DMQR_LIB_PATH=$L DMQR_NO_LOOKAHEAD=1 timeout 200 python tools/ab_time.py 8192 2 2>&1 | sed "s/^/$v serial /"
done; done
for v in base prev; do
  if [ $v = base ]; then L=""; else L=_ab/$v.so; fi
  DMQR_LIB_PATH=$L timeout 300 python tools/ab_time.py 16384 1 cfg5 2>&1 | sed "s/^/$v /"
done
