#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "graph or config5 or warm or tonal" > gpurun_out/pytest_guc.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_guc.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo done
