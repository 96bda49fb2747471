for v in base c6e noguard; do
  if [ $v = base ]; then L=""; else L=_ab/$v.so; fi
  DMQR_LIB_PATH=$L timeout 300 python tools/qrp_timing.py 2048 4096 2>&1 | sed "s/^/$v /"
done
N=/usr/local/cuda/bin/ncu
timeout 600 $N --set full --clock-control none --import-source on -k regex:k_spare -s 40 -c 3 -o gpurun_out/ncu15_spare python tools/ab_time.py 4096 0 > gpurun_out/ncu15_spare.log 2>&1
timeout 600 $N --set full --clock-control none --import-source on -k regex:"k_swap|k_gram|k_panel_cq|k_trail_w|k_select" -s 80 -c 7 -o gpurun_out/ncu15_step python tools/ab_time.py 4096 0 > gpurun_out/ncu15_step.log 2>&1
timeout 600 $N --set full --clock-control none --import-source on -k regex:k_qp3 -s 3 -c 1 -o gpurun_out/ncu15_qp3 python tools/qrp_timing.py 2048 > gpurun_out/ncu15_qp3.log 2>&1
