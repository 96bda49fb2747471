#!/bin/bash
# Run a command; if its log stops growing for 20 s, attach cuda-gdb and list the
# resident kernels / blocks / warps, then kill it.   tools/hang_watch.sh LOG -- cmd...
LOG=$1; shift; shift
"$@" > "$LOG" 2>&1 &
PID=$!
while kill -0 $PID 2>/dev/null; do
  sleep 5
  age=$(( $(date +%s) - $(stat -c %Y "$LOG") ))
  if [ $age -gt 40 ]; then
    echo "=== stalled for ${age}s: attaching cuda-gdb" >> "$LOG"
    timeout 180 /usr/local/cuda/bin/cuda-gdb -p $PID -batch -ex "info cuda kernels" -ex "info cuda blocks" \
      -ex "info cuda warps" -ex "thread apply all bt 8" >> "$LOG.gdb" 2>&1
    kill -9 $PID
    break
  fi
done
wait $PID; echo "exit $?" >> "$LOG"
