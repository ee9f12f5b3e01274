#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
FEMI_RASTER_MINB=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
echo done
