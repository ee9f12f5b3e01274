#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; rm -f gpurun_out/bench_sg*.json
for rep in 1 2; do
for G in 1 0; do
for B in 32 64; do
FEMI_SMEM_GATHER=$G FEMI_BAND=$B timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_sg${G}_b${B}_$rep.json 2>/dev/null
done; done; done
FEMI_LOOP_PROF=1 FEMI_BAND=64 timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e > /dev/null 2> gpurun_out/loopprof.err
echo done
