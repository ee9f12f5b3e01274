#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for case in c1 c2 graph dmulti tonal; do
    if [ "$tool" = "racecheck" ] && [ "$case" = "tonal" ]; then continue; fi
    timeout 900 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_cases.py $case \
      > gpurun_out/san/${tool}_${case}.log 2>&1
    echo "$tool $case rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san/${tool}_${case}.log | tail -1)" >> gpurun_out/san/summary.txt
  done
done
echo done
