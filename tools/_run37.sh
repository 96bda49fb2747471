N=/usr/local/cuda/bin/ncu
timeout 600 $N --set full --clock-control none --import-source on -k regex:"k_trail_w|k_gram_finish|k_select|k_swap|k_gram$" -s 200 -c 5 -o gpurun_out/ncu37_w python tools/ab_time.py 4096 0 > gpurun_out/ncu37_w.log 2>&1
tail -3 gpurun_out/ncu37_w.log
