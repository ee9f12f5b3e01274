#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "densify or config3 or warm or colour" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_c3i.json 2> gpurun_out/bench_c3i.err
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --rebuild-mesh > gpurun_out/bench_c3r.json 2> gpurun_out/bench_c3r.err
echo done
