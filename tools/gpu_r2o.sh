#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_o.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_o.log
FEMI_TONAL_PROF=1 timeout 600 python bench.py --config 4 --steps 3 --warmup 2 > gpurun_out/bench_o4.json 2> gpurun_out/bench_o4.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_o5.json 2> gpurun_out/bench_o5.err
echo done
