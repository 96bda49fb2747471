# compute-sanitizer (one tool at a time, small shapes) + ncu of the norm kernels
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san_memcheck.log
timeout 900 $S --tool racecheck --print-limit 20 python tools/sanitize_cases.py quick > gpurun_out/san_racecheck.log 2>&1; echo "exit $?" >> gpurun_out/san_racecheck.log
timeout 900 $S --tool synccheck --print-limit 20 python tools/sanitize_cases.py quick > gpurun_out/san_synccheck.log 2>&1; echo "exit $?" >> gpurun_out/san_synccheck.log
N=/usr/local/cuda/bin/ncu
timeout 600 $N --set full --clock-control none -k regex:"k_colnorms_init|k_guard_norms" -c 6 -o gpurun_out/ncu_norms_cfg2 python tools/ab_time.py 4096 1 > gpurun_out/ncu_norms_cfg2.log 2>&1
timeout 600 $N --set full --clock-control none -k regex:"k_colnorms_init|k_downdate|k_gnorm_part|k_gnorm_fin" -c 8 -o gpurun_out/ncu_norms_cfg4 python tools/ab_time.py 1024 1 cfg4 > gpurun_out/ncu_norms_cfg4.log 2>&1
ls -la gpurun_out
