timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest14.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest14.log
timeout 900 python bench.py > gpurun_out/bench14.log 2>&1; echo "bench exit $?" >> gpurun_out/bench14.log
N=/usr/local/cuda/bin/ncu
timeout 600 $N --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches14.csv python bench.py --steps 1 --warmup 3 --no-extra --no-cpu > gpurun_out/ncu14_launch.log 2>&1
timeout 600 $N --set full --clock-control none --import-source on -k regex:k_spare -s 40 -c 3 -o gpurun_out/ncu14_spare python tools/ab_time.py 4096 0 > gpurun_out/ncu14_spare.log 2>&1
timeout 600 $N --set full --clock-control none --import-source on -k regex:"k_swap|k_gram$|k_gram\b|k_panel_cq|k_trail_w|k_select|k_gram_finish" -s 80 -c 7 -o gpurun_out/ncu14_step python tools/ab_time.py 4096 0 > gpurun_out/ncu14_step.log 2>&1
