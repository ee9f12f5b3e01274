#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tonal --steps 5 --warmup 3 > gpurun_out/kb.json 2> gpurun_out/kbench.err
echo done
