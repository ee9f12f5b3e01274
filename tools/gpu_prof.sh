#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --config 2 --steps 1 --warmup 1"
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cgr" -s 1 -c 1 -o gpurun_out/prof_cgr $CMD > gpurun_out/prof_cgr.log 2>&1
echo done
