#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_raster" -s 3 -c 1 -o gpurun_out/prof_raster3 -f $CMD > gpurun_out/prof_raster3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
echo done
