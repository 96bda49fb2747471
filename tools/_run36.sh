timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused_step_tail or schedule_switches or lookahead_matches or fallback or pmode or streamed" 2>&1 | tail -5
for a in 4096 8192 cfg5:4096; do
  timeout 300 python tools/ab_equal.py $a 2>&1 | tail -1
  timeout 300 python tools/ab_equal.py $a DMQR_NO_FUSED_TAIL=1 2>&1 | tail -1
done
python tools/timeline.py 4096 > gpurun_out/r36_timeline.txt 2>&1; tail -12 gpurun_out/r36_timeline.txt
