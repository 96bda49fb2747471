#!/bin/bash
# The round's profiling pass, run on the GPU box (gpurun -- 'bash tools/profile_round.sh TAG'):
# a plain bench first (its numbers are the ones reported), then the ncu launch list of the same
# command, k_spare's DRAM traffic over one factorization, `--set full` captures of k_spare and of
# one step's kernels, the device timeline and the panel's phase clocks.  Everything lands in
# gpurun_out/ under TAG; tools/launch_summary.py, tools/ncu_table.py and tools/spare_traffic.py
# turn the captures into the tables committed under profiles/.
TAG=${1:-rXX}
N=/usr/local/cuda/bin/ncu
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench exit $?"; tail -c 300 $O/${TAG}_bench.err
timeout 900 $N --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > $O/${TAG}_ncu_l.log 2>&1; echo "launch list exit $?"
timeout 900 $N --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__ops_path_tensor_src_fp64.sum \
  --clock-control none -k regex:k_spare --csv --log-file $O/${TAG}_spare_traffic.csv python tools/ab_time.py 4096 0 > $O/${TAG}_ncu_t.log 2>&1; echo "traffic exit $?"
timeout 900 $N --set full --clock-control none --import-source on -k regex:"k_spare" -s 8 -c 2 -o $O/${TAG}_ncu_spare \
  python tools/ab_time.py 4096 0 > $O/${TAG}_ncu_spare.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on -k regex:"k_trail_w|k_tail|k_panel_cq|k_swap|k_gram|k_select" \
  -s 210 -c 7 -o $O/${TAG}_ncu_step python tools/ab_time.py 4096 0 > $O/${TAG}_ncu_step.log 2>&1
python tools/timeline.py 4096 > $O/${TAG}_timeline.txt 2>&1
python tools/cq_clocks.py 4096 2>&1 | tail -2 | head -1
