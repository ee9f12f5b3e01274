#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "warm or config3" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 3 --steps 3 --warmup 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config 3 --steps 3 --warmup 1 --warm > gpurun_out/bench_c3w.json 2> gpurun_out/bench_c3w.err
timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --n 30 > gpurun_out/bench_c3n.json 2> gpurun_out/bench_c3n.err
timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --n 30 --warm > gpurun_out/bench_c3nw.json 2> gpurun_out/bench_c3nw.err
echo done
