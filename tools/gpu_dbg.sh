#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "graph or config5 or warm or tonal or max" > gpurun_out/pytest_gu2.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gu2.log
for rep in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_gu2_$rep.json 2>/dev/null
done
FEMI_LOOP_PROF=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-tonal > /dev/null 2> gpurun_out/loop_gu2.err
echo done
