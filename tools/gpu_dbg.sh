#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FEMI_TONAL_PROF=1 timeout 300 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/bench_c4p.json 2> gpurun_out/bench_c4p.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 1 --warmup 0 > gpurun_out/ncu_c4.log 2>&1
echo done
