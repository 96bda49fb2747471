# where the time goes at 8192^2 / 16384^2 (serial schedule) + ncu on the trailing kernels
timeout 300 python tools/cfg_timing.py cfg2 8192 2>&1 | tail -1
timeout 600 python tools/cfg_timing.py cfg2 16384 2>&1 | tail -1
N=/usr/local/cuda/bin/ncu
timeout 900 $N --set full --clock-control none --import-source on -k regex:"k_trail_a|k_trail_b" -s 20 -c 4 -o gpurun_out/ncu31_trail python tools/ab_time.py 8192 0 > gpurun_out/ncu31_trail.log 2>&1
timeout 600 $N --metrics gpu__time_duration.sum --clock-control none -s 200 -c 600 --csv --log-file gpurun_out/launches31_8192.csv python tools/ab_time.py 8192 0 > gpurun_out/ncu31_l.log 2>&1
ls -la gpurun_out/
