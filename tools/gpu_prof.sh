#!/bin/bash
# ncu --set full captures of the solver body kernels (standalone launches via FEMI_PCG_KBENCH)
# and the raster kernels, C5 workload. Each ncu runs only after the same command exited 0.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
export FEMI_PCG_KBENCH=1
timeout 600 $CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:"k_gp" -s 20 -c 1 -o gpurun_out/prof_gp $CMD > gpurun_out/prof_gp.log 2>&1
timeout 900 $NCU -k regex:"k_gs" -s 20 -c 1 -o gpurun_out/prof_gs $CMD > gpurun_out/prof_gs.log 2>&1
timeout 900 $NCU -k regex:"k_gu" -s 20 -c 1 -o gpurun_out/prof_gu $CMD > gpurun_out/prof_gu.log 2>&1
unset FEMI_PCG_KBENCH
timeout 900 $NCU -k regex:"k_px_values|k_tri_reduce" -s 4 -c 2 -o gpurun_out/prof_raster $CMD > gpurun_out/prof_raster.log 2>&1
echo done
