#!/bin/bash
# standalone body kernels (FEMI_PCG_KBENCH) + ncu --set full of one k_gu and one k_gt
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal"
FEMI_PCG_KBENCH=1 timeout 600 $CMD > gpurun_out/kbench.json 2> gpurun_out/kbench.err || { echo "plain run failed"; exit 1; }
FEMI_PCG_KBENCH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gu|k_gt" -s 8 -c 2 \
  -o gpurun_out/prof_body $CMD > gpurun_out/prof_body.log 2>&1
echo done
