#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "tonal or config4 or smoke" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
for rep in 1 2; do FEMI_TONAL_PROF=1 timeout 300 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/bench_c4_$rep.json 2> gpurun_out/bench_c4_$rep.err; done
echo done
