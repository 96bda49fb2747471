N=/usr/local/cuda/bin/ncu
timeout 900 python bench.py > gpurun_out/r50_bench.json 2> gpurun_out/r50_bench.err; echo "bench exit $?"; tail -c 300 gpurun_out/r50_bench.err
timeout 900 $N --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r50_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > gpurun_out/r50_ncu_l.log 2>&1; echo "launch list exit $?"
timeout 900 $N --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__ops_path_tensor_src_fp64.sum --clock-control none -k regex:k_spare --csv --log-file gpurun_out/spare_traffic.csv python tools/ab_time.py 4096 0 > gpurun_out/r50_ncu_t.log 2>&1; echo "traffic exit $?"
timeout 900 $N --set full --clock-control none --import-source on -k regex:"k_spare" -s 8 -c 2 -o gpurun_out/ncu50_spare python tools/ab_time.py 4096 0 > gpurun_out/ncu50_spare.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on -k regex:"k_trail_w|k_tail|k_panel_cq|k_swap|k_gram|k_select" -s 210 -c 7 -o gpurun_out/ncu50_step python tools/ab_time.py 4096 0 > gpurun_out/ncu50_step.log 2>&1
python tools/timeline.py 4096 > gpurun_out/r50_timeline.txt 2>&1
python tools/cq_clocks.py 4096 2>&1 | tail -2 | head -1
