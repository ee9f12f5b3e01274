#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_r4_$rep.json 2>/dev/null
done
cp paper_2105_01586_b200/libfemi.so /tmp/libfemi_base.so; cp tools/_tmp/libfemi_v.so paper_2105_01586_b200/libfemi.so; touch paper_2105_01586_b200/libfemi.so
for rep in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tonal > gpurun_out/bench_r5_$rep.json 2>/dev/null
done
timeout 600 python -m pytest tests -m gpu -x -q -k "config1 or inpaint or max" > gpurun_out/pytest_r5.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r5.log
echo done
