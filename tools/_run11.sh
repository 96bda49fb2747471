for rep in 1 2; do
for v in base notma mlub notma_mlub; do
  if [ $v = base ]; then L=""; else L=_ab/$v.so; fi
  DMQR_LIB_PATH=$L timeout 200 python tools/ab_time.py 4096 5 2>&1 | sed "s/^/$v /"
done; done
for v in base mlub; do
  if [ $v = base ]; then L=""; else L=_ab/$v.so; fi
  for cta in 0 1; do DMQR_LIB_PATH=$L timeout 100 python tools/cq_clocks.py 4096 $cta 2>&1 | sed "s/^/$v /"; done
done
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest11.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest11.log
