for a in 3000 4096 8192; do
  timeout 120 python tools/ab_equal.py $a DMQR_NO_LOOKAHEAD=1 DMQR_NO_TB3=1 2>&1 | tail -1
  timeout 120 python tools/ab_equal.py $a DMQR_NO_LOOKAHEAD=1 2>&1 | tail -1
  timeout 120 python tools/ab_equal.py $a DMQR_NO_TB3=1 2>&1 | tail -1
  timeout 120 python tools/ab_equal.py $a 2>&1 | tail -1
done
timeout 200 python tools/ab_equal.py 16384 DMQR_NO_TB3=1 2>&1 | tail -1
timeout 200 python tools/ab_equal.py 16384 2>&1 | tail -1
timeout 200 python tools/ab_equal.py 16384 DMQR_FORCE_LOOKAHEAD=1 2>&1 | tail -1
