#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_lx.json 2> gpurun_out/bench_lx.err
FEMI_LOOP_PROF=1 timeout 300 python bench.py --steps 2 --warmup 1 > /dev/null 2> gpurun_out/loopprof.err
echo done
