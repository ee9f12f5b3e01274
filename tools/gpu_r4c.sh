#!/bin/bash
# per-kernel durations of one C4 resident solve (ncu launch list) and of the C4 tonal bench
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/r4c; mkdir -p $O
timeout 300 python tools/diag_cgr.py 4 1 > $O/plain.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4solve.csv python tools/diag_cgr.py 4 1 > $O/ncu1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 2000 --log-file $O/launches_c4tonal.csv python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu2.log 2>&1
echo done
