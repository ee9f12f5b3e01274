#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_h5.json 2> gpurun_out/bench_h5.err
timeout 900 python -m pytest tests -m gpu -q -x -k "raster or inpaint or config or colour or c5_legs or max_image or tonal or x0 or graph" > gpurun_out/pytest_h.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_h.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_raster_grp" -s 3 -c 1 -o gpurun_out/prof_raster7 -f $CMD > gpurun_out/prof_raster7.log 2>&1
echo done
