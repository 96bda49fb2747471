timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused_step_tail or schedule_switches or lookahead_matches or fallback or pmode or golden" 2>&1 | tail -3
for a in 4096 8192; do
  timeout 300 python tools/ab_equal.py $a 2>&1 | tail -1
done
python tools/timeline.py 4096 > gpurun_out/r39_timeline.txt 2>&1; tail -22 gpurun_out/r39_timeline.txt
