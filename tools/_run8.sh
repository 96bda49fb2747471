set -x
for v in r16n3 r24n3 r32n2; do DMQR_LIB_PATH=_ab/$v.so timeout 200 python tools/ab_time.py 4096 5 2>&1 | sed "s/^/$v /"; done
timeout 200 python tools/ab_time.py 4096 5 2>&1 | sed "s/^/base /"
for v in r16n3 r24n3 r32n2; do DMQR_LIB_PATH=_ab/$v.so timeout 300 python tools/ab_time.py 8192 2 2>&1 | sed "s/^/$v /"; done
timeout 300 python tools/ab_time.py 8192 2 2>&1 | sed "s/^/base /"
DMQR_FORCE_LOOKAHEAD=1 timeout 300 python tools/ab_time.py 8192 2 2>&1 | sed "s/^/base-LA /"
timeout 600 python tools/ab_time.py 16384 1 2>&1 | sed "s/^/base /"
DMQR_FORCE_LOOKAHEAD=1 timeout 600 python tools/ab_time.py 16384 1 2>&1 | sed "s/^/base-LA /"
timeout 300 python tools/cfg_timeline.py cfg2 2>&1
timeout 300 python tools/small_clocks.py 2>&1
