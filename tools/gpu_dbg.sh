#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for rep in 1; do
timeout 300 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/bench_c2_$rep.json 2>/dev/null
timeout 300 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/bench_c4_$rep.json 2>/dev/null
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_$rep.json 2>/dev/null
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_c3_$rep.json 2>/dev/null
done
echo done
