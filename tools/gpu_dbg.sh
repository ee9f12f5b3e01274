#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in 1 2; do
FEMI_FUSED=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_fused_$rep.json 2>/dev/null
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_base_$rep.json 2>/dev/null
done
echo done
