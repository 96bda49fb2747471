N=/usr/local/cuda/bin/ncu
for v in "" NOMMA NOLOADC NOSTORE NOLS; do
  L=""; [ -n "$v" ] && L=_ab/$v.so
  DMQR_LIB_PATH=$L DMQR_NO_LOOKAHEAD=1 DMQR_NO_TB2=1 timeout 300 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_trail_b|k_trail_a" -c 2 --csv python tools/ab_time.py 8192 0 2>/dev/null | grep -v "^==" | awk -F'","' -v v="$v" 'NR>1{print v, $5, $(NF-2), $(NF)}' | tr -d '"'
done
