#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for G in 1184 592 888; do
FEMI_GUM_CTAS=$G timeout 300 python bench.py --config 6 --steps 5 --warmup 3 > gpurun_out/bench_gum_$G.json 2>/dev/null
done
echo done
