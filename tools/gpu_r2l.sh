#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_f.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_f.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_f5.json 2> gpurun_out/bench_f5.err
FEMI_L2POL=3 FEMI_DEBUG=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_p3.json 2> gpurun_out/bench_p3.err
FEMI_L2POL=2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_p2.json 2> gpurun_out/bench_p2.err
FEMI_L2POL=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tonal > gpurun_out/bench_p1.json 2> gpurun_out/bench_p1.err
for c in 2 3 4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_f$c.json 2> gpurun_out/bench_f$c.err; done
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f1.json 2> gpurun_out/bench_f1.err
echo done
