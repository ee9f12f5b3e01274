#!/bin/bash
# session re-entry check: full GPU suite + C5 bench + loop timeline on HEAD
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/r3a
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r3a/bench_c5.json 2> gpurun_out/r3a/bench_c5.err
FEMI_LOOP_PROF=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/r3a/loop.json 2> gpurun_out/r3a/loop.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3a/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3a/pytest_gpu.log
echo done
