#!/bin/bash
# quick GPU check: GPU tests (optionally filtered by $PYTEST_K) + C5 bench (+ extra bench args)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
if [ -n "$BENCH2" ]; then timeout 300 python bench.py $BENCH2 > gpurun_out/bench_q2.json 2> gpurun_out/bench_q2.err; fi
echo done
