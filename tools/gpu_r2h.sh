#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "tonal_channels" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_tc.log
FEMI_TONAL_PROF=1 timeout 600 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
FEMI_TONAL_PROF=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5t.json 2> gpurun_out/bench_c5t.err
timeout 900 python bench.py --config 6 --steps 3 --warmup 2 > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err
echo done
