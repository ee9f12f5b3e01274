#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
FEMI_LIB=libfemi_check.so timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_check.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_check.log
echo done
