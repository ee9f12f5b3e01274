#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "colour" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 6 --steps 3 --warmup 2 > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err
echo done
