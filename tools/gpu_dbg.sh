#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_final.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_final.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo done
