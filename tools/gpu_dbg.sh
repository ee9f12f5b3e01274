#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in 2 3 4; do FEMI_PCG_TIMERS=1 timeout 300 python bench.py --config $c --steps 3 --warmup 1 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python -m pytest tests -m gpu -x -q -k "config2 or config3 or tonal or config1 or small" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
echo done
