#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python tools/diag_solve_overhead.py > gpurun_out/diag_ovh.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_g5.json 2> gpurun_out/bench_g5.err
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err
timeout 900 python -m pytest tests -m gpu -q -x -k "x0 or raster or inpaint or config" > gpurun_out/pytest_g.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_g.log
echo done
