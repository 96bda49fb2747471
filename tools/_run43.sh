N=/usr/local/cuda/bin/ncu
DMQR_NO_LOOKAHEAD=1 timeout 600 $N --set full --clock-control none --import-source on -k regex:"k_trail_b3" -s 1 -c 2 -o gpurun_out/ncu43_b3 python tools/ab_time.py 8192 0 > gpurun_out/ncu43_b3.log 2>&1
DMQR_NO_LOOKAHEAD=1 DMQR_NO_TB3=1 timeout 600 $N --set full --clock-control none --import-source on -k regex:"k_trail_b" -s 1 -c 2 -o gpurun_out/ncu43_b python tools/ab_time.py 8192 0 > gpurun_out/ncu43_b.log 2>&1
