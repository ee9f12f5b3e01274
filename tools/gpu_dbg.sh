#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FEMI_FUSED2=1 timeout 120 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_f2_try.json 2> gpurun_out/bench_f2_try.err; echo "rc $?" >> gpurun_out/bench_f2_try.err
if grep -q "rc 0" gpurun_out/bench_f2_try.err; then
for rep in 1 2; do
FEMI_FUSED2=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_f2_$rep.json 2>/dev/null
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_f0_$rep.json 2>/dev/null
done
FEMI_FUSED2=1 timeout 600 python -m pytest tests -m gpu -x -q -k "graph or config5 or warm" > gpurun_out/pytest_f2.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_f2.log
fi
echo done
