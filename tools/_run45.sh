timeout 120 python tools/ab_equal.py 8192 DMQR_NO_LOOKAHEAD=1 DMQR_NO_TB3=1 2>&1 | tail -1
timeout 120 python tools/ab_equal.py 8192 DMQR_NO_LOOKAHEAD=1 2>&1 | tail -1
timeout 200 python tools/ab_equal.py 16384 DMQR_NO_TB3=1 2>&1 | tail -1
timeout 200 python tools/ab_equal.py 16384 2>&1 | tail -1
timeout 200 python tools/ab_equal.py cfg4:1024 DMQR_NO_TB3=1 2>&1 | tail -1
timeout 200 python tools/ab_equal.py cfg4:1024 2>&1 | tail -1
timeout 200 python tools/ab_equal.py cfg5:16384 DMQR_NO_TB3=1 2>&1 | tail -1
timeout 200 python tools/ab_equal.py cfg5:16384 2>&1 | tail -1
