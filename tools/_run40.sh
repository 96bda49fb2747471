timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r40_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r40_gputest.log
tail -4 gpurun_out/r40_gputest.log
timeout 900 python bench.py > gpurun_out/r40_bench.json 2> gpurun_out/r40_bench.err; echo "bench exit $?"
tail -c 400 gpurun_out/r40_bench.err
