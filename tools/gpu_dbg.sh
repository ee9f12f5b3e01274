#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
(timeout 120 python tools/asm_bench.py 3; timeout 120 python tools/asm_bench.py 4) > gpurun_out/asm.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_c3s.json 2> gpurun_out/bench_c3s.err
echo done
