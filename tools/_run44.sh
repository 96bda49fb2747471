for a in 3000 8192; do
  timeout 120 python tools/ab_equal.py $a DMQR_NO_LOOKAHEAD=1 DMQR_NO_TB3=1 2>&1 | tail -1
  timeout 120 python tools/ab_equal.py $a DMQR_NO_LOOKAHEAD=1 2>&1 | tail -1
  timeout 120 python tools/ab_equal.py $a DMQR_NO_TB3=1 2>&1 | tail -1
  timeout 120 python tools/ab_equal.py $a 2>&1 | tail -1
done
timeout 120 python tools/ab_equal.py 4096 2>&1 | tail -1
timeout 200 python tools/ab_equal.py 16384 2>&1 | tail -1
timeout 200 python tools/ab_equal.py 16384 DMQR_FORCE_LOOKAHEAD=1 2>&1 | tail -1
N=/usr/local/cuda/bin/ncu
DMQR_NO_LOOKAHEAD=1 timeout 600 $N --set full --clock-control none --import-source on -k regex:"k_trail_b3" -s 1 -c 2 -o gpurun_out/ncu44_b3 python tools/ab_time.py 8192 0 > gpurun_out/ncu44_b3.log 2>&1
