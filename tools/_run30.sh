# round-2 re-entry: full GPU suite + bench at HEAD
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r30_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r30_gputest.log
tail -5 gpurun_out/r30_gputest.log
timeout 900 python bench.py > gpurun_out/r30_bench.json 2> gpurun_out/r30_bench.err; echo "bench exit $?"
tail -c 600 gpurun_out/r30_bench.err
python tools/timeline.py 4096 > gpurun_out/r30_timeline.txt 2>&1; tail -20 gpurun_out/r30_timeline.txt
