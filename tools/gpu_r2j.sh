#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --config 3 --steps 3 --warmup 2 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
FEMI_ASM_PROF=1 FEMI_MESH_PROF=1 timeout 600 python bench.py --config 3 --steps 1 --warmup 1 > gpurun_out/bench_c3p.json 2> gpurun_out/bench_c3p.err
timeout 1200 python bench.py --config 3 --steps 2 --warmup 1 --n 100 --warm > gpurun_out/bench_c3n100.json 2> gpurun_out/bench_c3n100.err
timeout 900 python -m pytest tests -m gpu -q -x -k "config3 or densify or config2 or config1" > gpurun_out/pytest_s.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_s.log
echo done
