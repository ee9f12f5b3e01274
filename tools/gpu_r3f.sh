#!/bin/bash
# C3 host stage split at pool sizes 16 / 8 / 4 / 1
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/r3f
for t in 16 8 4 1; do FEMI_POOL_THREADS=$t timeout 300 python tools/diag_c3_stages.py 3 > gpurun_out/r3f/stages_$t.txt 2>&1; done
echo done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_raster_grp" -s 3 -c 1 -o gpurun_out/r3f/prof_raster -f $CMD > gpurun_out/r3f/prof_raster.log 2>&1
echo done2
