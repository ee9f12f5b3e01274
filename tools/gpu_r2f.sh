#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
FEMI_FUSED=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_q0.json 2> gpurun_out/bench_q0.err
timeout 900 python -m pytest tests -m gpu -q -x -k "graph or c5_legs or colour or max_image" > gpurun_out/pytest_gf.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gf.log
echo done
