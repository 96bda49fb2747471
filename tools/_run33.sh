for a in 3000 4096 8192; do
  for L in _ab/prev.so ""; do
    DMQR_LIB_PATH=$L timeout 300 python tools/ab_equal.py $a 2>&1 | tail -1
    DMQR_LIB_PATH=$L timeout 300 python tools/ab_equal.py $a DMQR_NO_LOOKAHEAD=1 DMQR_NO_TB2=1 2>&1 | tail -1
  done
  timeout 300 python tools/ab_equal.py $a DMQR_NO_LOOKAHEAD=1 2>&1 | tail -1
done
for L in _ab/prev.so ""; do
  DMQR_LIB_PATH=$L timeout 300 python tools/ab_equal.py 16384 DMQR_NO_TB2=1 2>&1 | tail -1
  DMQR_LIB_PATH=$L timeout 300 python tools/ab_equal.py cfg4:1024 DMQR_NO_TB2=1 2>&1 | tail -1
  DMQR_LIB_PATH=$L timeout 300 python tools/ab_equal.py cfg5:4096 DMQR_NO_TB2=1 2>&1 | tail -1
done
timeout 300 python tools/ab_equal.py 16384 2>&1 | tail -1
