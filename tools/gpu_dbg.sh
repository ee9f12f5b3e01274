#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_c3s.json 2> gpurun_out/bench_c3s.err
FEMI_SEL_MULTI=1 timeout 300 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_c3m.json 2> gpurun_out/bench_c3m.err
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --warm > gpurun_out/bench_c3w.json 2> gpurun_out/bench_c3w.err
echo done
