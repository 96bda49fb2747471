for rep in 1 2 3; do
for v in base notma tgram tswap; do
  if [ $v = base ]; then L=""; else L=_ab/$v.so; fi
  DMQR_LIB_PATH=$L timeout 200 python tools/ab_time.py 4096 5 2>&1 | sed "s/^/$v /"
done; done
timeout 600 python tools/ab_time.py 16384 1 cfg5 2>&1 | sed "s/^/serial /"
DMQR_FORCE_LOOKAHEAD=1 timeout 600 python tools/ab_time.py 16384 1 cfg5 2>&1 | sed "s/^/LA /"
timeout 600 python tools/ab_time.py 1024 3 cfg4 2>&1 | sed "s/^/serial /"
DMQR_FORCE_LOOKAHEAD=1 timeout 600 python tools/ab_time.py 1024 3 cfg4 2>&1 | sed "s/^/LA /"
