timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused_step_tail or schedule_switches or lookahead_matches or fallback" 2>&1 | tail -3
for a in 4096 8192 cfg4:1024; do
  timeout 300 python tools/ab_equal.py $a 2>&1 | tail -1
done
DMQR_LIB_PATH=_ab/prev.so timeout 300 python tools/ab_equal.py cfg4:1024 2>&1 | tail -1
python tools/timeline.py 4096 > gpurun_out/r38_timeline.txt 2>&1; tail -12 gpurun_out/r38_timeline.txt
