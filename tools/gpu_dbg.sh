#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in 1 2; do
for P in 0 2 6; do
FEMI_PDL_PRE=$P timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_pre${P}_$rep.json 2>/dev/null
done
FEMI_NO_PDL=1 timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_nopdl_$rep.json 2>/dev/null
done
echo done
