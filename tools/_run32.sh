timeout 900 python tools/tb2_check.py 3000 4096 8192 16384 2>&1 | grep -v Warning
N=/usr/local/cuda/bin/ncu
DMQR_NO_LOOKAHEAD=1 timeout 900 $N --set full --clock-control none --import-source on -k regex:"k_trail_a|k_trail_b" -s 20 -c 4 -o gpurun_out/ncu32_trail python tools/ab_time.py 8192 0 > gpurun_out/ncu32_trail.log 2>&1
