#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/bench_c2s.json 2> gpurun_out/bench_c2s.err
timeout 300 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/bench_c4s.json 2> gpurun_out/bench_c4s.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1s.json 2> gpurun_out/bench_c1s.err
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_c3s.json 2> gpurun_out/bench_c3s.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
echo done
