#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
timeout 600 $CMD > gpurun_out/plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_raster" -s 3 -c 1 -o gpurun_out/prof_raster2 -f $CMD > gpurun_out/prof_raster2.log 2>&1
echo done
