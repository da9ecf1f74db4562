#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of every kernel family on
# scaled-down configurations (tools/sanitize_case.py); logs under $1.
out=${1:-gpurun_out/sanitizer}
mkdir -p "$out"
for tool in memcheck racecheck synccheck; do
  for ci in 1 2 3 4; do
    compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_case.py $ci > "$out/${tool}_C$((ci+1)).log" 2>&1
    echo "$tool C$((ci+1)) rc=$?" | tee -a "$out/summary.txt"
  done
done
