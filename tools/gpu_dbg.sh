#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for pol in 0 1 2; do
FEMI_JDS_POLICY=$pol FEMI_PCG_KBENCH=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/kb_$pol.json 2> gpurun_out/kbench_$pol.err
FEMI_JDS_POLICY=$pol timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$pol.json 2> gpurun_out/bench_$pol.err
done
echo done
